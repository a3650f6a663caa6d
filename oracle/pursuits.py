"""Oracle greedy pursuits with the CG-based weighted LS step (fp64).  TEST INFRASTRUCTURE.

* OMP     — PAPER.md:243-257 (steps 1-4) and Algorithm 1 lines 01-10.
* SP      — named at P:84, P:221, P:574-576 (CG-SP); body not given in the
            paper, reconstructed per S:286-294 + SURVEY §8c.4 (reading R15).
* OMPR(l) — named at P:574-576 (CG-OMPR); body not given, reconstructed per
            S:296-304 + SURVEY §8c.5 (reading R16).
* CoSaMP  — named at P:84 among the greedy methods; body not
            given in the paper: the published CoSaMP iteration (Needell & Tropp) with
            the paper's CG as its LS step and this build's halting rule (reading R33).

Every least-squares step is `oracle.cg.cg` (Eq.(11)) warm-started from
the previous iterate (BASELINE.json; reading R9).  When the warm start is the
previous LS iterate on a superset-or-equal support, r0 = W A^T (y - A x0) is
exactly the correlation c already computed for detection (b - H x0 =
(A^T y - A^T A x0)[S] = (A^T r)[S]); after an index is removed, r0 = b - H x0 is
recomputed with one extra H apply.

Selection semantics (reading R12/R32): top-K of |v| with ties to
the lowest index; argmax excludes the current support.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .cg import cg, CONVERGED
from .dense import lstsq_on_support

# termination codes for pursuits (mirror cs_term in include/cs.h by value only)
T_DONE, T_ITER_CAP, T_SUPPORT_FIXED, T_RESID_ROSE = 0, 1, 3, 4


@dataclasses.dataclass
class PursuitResult:
    support: np.ndarray      # sorted int64[K]
    x: np.ndarray            # values on support
    s_hat: np.ndarray        # dense float64[N]
    outer_iters: int
    cg_iters: int
    resid_norm: float        # ||y - A s_hat||
    termination: int
    resid_history: list


def topk(v: np.ndarray, K: int, allowed: Optional[np.ndarray] = None) -> np.ndarray:
    """Indices of the K largest v (ties -> lowest index), returned sorted ascending.

    `allowed` is a boolean mask; disallowed entries are never chosen."""
    idx = np.arange(v.size)
    if allowed is not None:
        idx = idx[allowed]
    vals = v[idx]
    order = np.lexsort((idx, -vals))          # primary: -v ascending, secondary: index
    return np.sort(idx[order[:K]])


def _scatter(N, S, x):
    xt = np.zeros(N)
    xt[S] = x
    return xt


class _LS:
    """The LS step: 'cg' = the paper's CG (default), 'lstsq' = dense oracle backend."""

    def __init__(self, op, y, c0, solver, tol, cg_cap):
        self.op, self.y, self.c0 = op, y, c0
        self.solver, self.tol, self.cg_cap = solver, tol, cg_cap
        self.iters = 0

    def __call__(self, S, x0=None, r0=None):
        if self.solver == "lstsq":
            return lstsq_on_support(self.op, S, self.y)
        res = cg(self.op, S, self.c0, x0=x0, r0=r0, tol=self.tol,
                 cap=None if not self.cg_cap else self.cg_cap)
        self.iters += res.iters
        return res.x


def omp(op, y, K, tol=1e-10, solver="cg", cg_cap=0) -> PursuitResult:
    """Algorithm 1: exactly K outer iterations (reading R13)."""
    y = np.asarray(y, dtype=np.float64)
    N = op.N
    c0 = op.adjoint(y)                         # s_0 = A^T y, used as b source
    ls = _LS(op, y, c0, solver, tol, cg_cap)
    r = y.copy()                               # r_0 = y
    S = np.zeros(0, dtype=np.int64)
    x = np.zeros(0)
    hist = []
    for i in range(K):                         # line 02
        c = op.adjoint(r)                      # line 03: A^T r_{i-1}
        a = np.abs(c)
        a[S] = -1.0                            # exclude S (R12)
        t = int(np.argmax(a))                  # Eq.(6); first max = lowest index
        pos = int(np.searchsorted(S, t))
        S = np.insert(S, pos, t)               # line 04
        x = np.insert(x, pos, 0.0)
        x = ls(S, x0=x, r0=c[S])               # line 06 (warm start, free r0)
        r = y - op.apply(_scatter(N, S, x))    # line 07
        hist.append(float(np.linalg.norm(r)))
    return PursuitResult(S, x, _scatter(N, S, x), K, ls.iters,
                         float(np.linalg.norm(r)), T_DONE, hist)


def sp(op, y, K, tol=1e-10, max_outer=30, solver="cg", cg_cap=0) -> PursuitResult:
    """CG-SP (body per S:289 and SURVEY §8c.4)."""
    y = np.asarray(y, dtype=np.float64)
    N = op.N
    c0 = op.adjoint(y)
    ls = _LS(op, y, c0, solver, tol, cg_cap)
    S = topk(np.abs(c0), K)
    x = ls(S, x0=None, r0=c0[S])
    r = y - op.apply(_scatter(N, S, x))
    rn = float(np.linalg.norm(r))
    hist = [rn]
    term, it = T_ITER_CAP, 0
    for it in range(1, max_outer + 1):
        c = op.adjoint(r)
        notS = np.ones(N, dtype=bool)
        notS[S] = False
        J = topk(np.abs(c), K, allowed=notS)
        T = np.union1d(S, J)
        xt = _scatter(N, S, x)
        xT = ls(T, x0=xt[T], r0=c[T])
        keep = np.zeros(N, dtype=bool)
        keep[T] = True
        dT = np.zeros(N)
        dT[T] = np.abs(xT)
        S2 = topk(dT, K, allowed=keep)
        if np.array_equal(S2, S):
            term = T_SUPPORT_FIXED
            break
        xT_dense = _scatter(N, T, xT)
        x2 = ls(S2, x0=xT_dense[S2], r0=None)
        r2 = y - op.apply(_scatter(N, S2, x2))
        rn2 = float(np.linalg.norm(r2))
        if rn2 >= rn:
            term = T_RESID_ROSE
            break
        S, x, r, rn = S2, x2, r2, rn2
        hist.append(rn)
    return PursuitResult(S, x, _scatter(N, S, x), it, ls.iters, rn, term, hist)


def ompr(op, y, K, tol=1e-10, l=1, eta=1.0, max_outer=0, solver="cg", cg_cap=0) -> PursuitResult:
    """CG-OMPR(l, eta) (body per S:299 and SURVEY §8c.5, R16, R31)."""
    y = np.asarray(y, dtype=np.float64)
    N = op.N
    max_outer = 2 * K if max_outer <= 0 else max_outer
    c0 = op.adjoint(y)
    ls = _LS(op, y, c0, solver, tol, cg_cap)
    S = topk(np.abs(c0), K)
    x = ls(S, x0=None, r0=c0[S])
    r = y - op.apply(_scatter(N, S, x))
    hist = [float(np.linalg.norm(r))]
    term, t = T_ITER_CAP, 0
    for t in range(1, max_outer + 1):
        c = op.adjoint(r)
        xt = _scatter(N, S, x)
        z = xt + eta * c
        notS = np.ones(N, dtype=bool)
        notS[S] = False
        J = topk(np.abs(z), l, allowed=notS)
        U = np.union1d(S, J)
        inU = np.zeros(N, dtype=bool)
        inU[U] = True
        S2 = topk(np.abs(z), K, allowed=inU)
        if np.array_equal(S2, S):
            term = T_SUPPORT_FIXED
            break
        x = ls(S2, x0=xt[S2], r0=None)
        S = S2
        r = y - op.apply(_scatter(N, S, x))
        hist.append(float(np.linalg.norm(r)))
    return PursuitResult(S, x, _scatter(N, S, x), t, ls.iters,
                         float(np.linalg.norm(r)), term, hist)


def cosamp(op, y, K, tol=1e-10, max_outer=30, solver="cg", cg_cap=0) -> PursuitResult:
    """CG-CoSaMP (named P:84; iteration per Needell & Tropp, reading R33).

    x = 0, S = {} ; repeat:  c = A^T (y - A x);  Omega = top-2K of |c| (all indices);
    T = Omega u S;  b_T = LS on T (CG, warm start x, free r0 = c[T]);  S' = top-K of
    |b_T| over T;  x' = b_T on S' (no second LS);  r' = y - A x'.
    Halting: ||r'|| >= ||r|| after the first iteration -> keep (S, x) (T_RESID_ROSE);
    otherwise accept (S', x') and stop if S' == S (T_SUPPORT_FIXED); max_outer -> cap."""
    y = np.asarray(y, dtype=np.float64)
    N = op.N
    c0 = op.adjoint(y)
    ls = _LS(op, y, c0, solver, tol, cg_cap)
    S = np.zeros(0, dtype=np.int64)
    x = np.zeros(0)
    c = c0                                         # A^T (y - A 0)
    rn = float(np.linalg.norm(y))
    hist = [rn]
    term, it = T_ITER_CAP, 0
    for it in range(1, max_outer + 1):
        Om = topk(np.abs(c), min(2 * K, N))
        T = np.union1d(S, Om)
        xT = ls(T, x0=_scatter(N, S, x)[T], r0=c[T])
        keep = np.zeros(N, dtype=bool)
        keep[T] = True
        dT = np.zeros(N)
        dT[T] = np.abs(xT)
        S2 = topk(dT, K, allowed=keep)
        x2 = _scatter(N, T, xT)[S2]
        r2 = y - op.apply(_scatter(N, S2, x2))
        rn2 = float(np.linalg.norm(r2))
        if it > 1 and rn2 >= rn:
            term = T_RESID_ROSE
            break
        fixed = np.array_equal(S2, S)
        S, x, rn = S2, x2, rn2
        hist.append(rn)
        if fixed:
            term = T_SUPPORT_FIXED
            break
        c = op.adjoint(r2)
    return PursuitResult(S, x, _scatter(N, S, x), it, ls.iters, rn, term, hist)


def recover(alg, op, y, K, **kw) -> PursuitResult:
    return {"omp": omp, "sp": sp, "ompr": ompr, "cosamp": cosamp}[alg](op, y, K, **kw)
