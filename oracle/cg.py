"""Oracle CG-based weighted least squares (fp64).  TEST INFRASTRUCTURE.

Algorithm 1, function CG, solving Eq.(11)
    W^T A^T A W theta = W^T A^T y
restricted to the support S (Theorem 5's reduced system, Eq.(12), P:526 — the
masked iterates equal the reduced ones, so we carry |S|-length
vectors; W_S is never materialised).

Readings: the loop condition is `while ||r_j|| > xi` (the
printed `<=` at P:462 is a typo, R6); xi is relative to ||b|| (R7); the solve
is warm-started at x0 (BASELINE.json, R9) with r0 = b - H x0 (or a caller-given
r0 that equals it, see pursuits.py); breakdown d^T H d <= 0 stops with
STAGNATION; the iteration cap is |S| + 50 (Thm 5 bound |S| plus slack,
R29).
"""
from __future__ import annotations

import dataclasses

import numpy as np

CONVERGED, ITER_CAP, STAGNATION = 0, 1, 2


@dataclasses.dataclass
class CgResult:
    x: np.ndarray          # solution on S (compact, |S|)
    iters: int             # j at exit
    resid: float           # ||r_j|| at exit (normal-equation residual)
    bnorm: float           # ||b||
    termination: int
    alphas: list
    betas: list
    rnorms: list


def support_H(op, S):
    """v -> (A^T A scatter_S(v))[S] = H restricted to S."""
    S = np.asarray(S, dtype=np.int64)

    def H(v):
        xt = np.zeros(op.N)
        xt[S] = v
        return op.adjoint(op.apply(xt))[S]
    return H


def cg(op, S, c0, x0=None, r0=None, tol=1e-10, cap=None, trace=False) -> CgResult:
    """Algorithm 1 lines 11-23 on support S.

    c0 = A^T y (so b = W^T A^T y restricted to S is c0[S], line 12).
    """
    S = np.asarray(S, dtype=np.int64)
    H = support_H(op, S)
    b = np.asarray(c0, dtype=np.float64)[S]                      # line 12
    x = np.zeros(S.size) if x0 is None else np.array(x0, dtype=np.float64)   # line 13 / warm start
    if r0 is not None:
        r = np.array(r0, dtype=np.float64)
    elif x0 is None:
        r = b.copy()                                              # line 13: r_0 = b
    else:
        r = b - H(x)
    d = r.copy()                                                  # line 13: d_0 = r_0
    rho = float(r @ r)
    bnorm = float(np.linalg.norm(b))
    cap = S.size + 50 if cap is None else cap
    j = 0                                                         # line 14
    term = CONVERGED
    alphas, betas, rnorms = [], [], [np.sqrt(rho)]
    while np.sqrt(rho) > tol * bnorm:                             # line 15 (R6, R7)
        if j >= cap:
            term = ITER_CAP
            break
        q = H(d)
        dq = float(d @ q)
        if dq <= 0.0:
            term = STAGNATION
            break
        alpha = rho / dq                                          # line 16
        x = x + alpha * d                                         # line 17
        r = r - alpha * q                                         # line 18
        rho_new = float(r @ r)
        beta = rho_new / rho                                      # line 19
        d = r + beta * d                                          # line 20
        rho = rho_new
        j += 1                                                    # line 21
        if trace:
            alphas.append(alpha)
            betas.append(beta)
            rnorms.append(np.sqrt(rho))
    return CgResult(x, j, float(np.sqrt(rho)), bnorm, term, alphas, betas, rnorms)


def reduced_cg(AS: np.ndarray, y: np.ndarray, tol=1e-13, cap=None) -> CgResult:
    """CG on the explicit reduced SPD system A_S^T A_S s = A_S^T y (Eq.(12)).

    Test-side pin for Theorem 5: the masked iteration above must follow this
    trace step for step."""
    G = AS.T @ AS
    b = AS.T @ y
    x = np.zeros(AS.shape[1])
    r = b.copy()
    d = r.copy()
    rho = float(r @ r)
    bnorm = float(np.linalg.norm(b))
    cap = AS.shape[1] + 50 if cap is None else cap
    j = 0
    alphas, betas, rnorms = [], [], [np.sqrt(rho)]
    term = CONVERGED
    while np.sqrt(rho) > tol * bnorm:
        if j >= cap:
            term = ITER_CAP
            break
        q = G @ d
        dq = float(d @ q)
        if dq <= 0:
            term = STAGNATION
            break
        alpha = rho / dq
        x = x + alpha * d
        r = r - alpha * q
        rho_new = float(r @ r)
        beta = rho_new / rho
        d = r + beta * d
        rho = rho_new
        j += 1
        alphas.append(alpha)
        betas.append(beta)
        rnorms.append(np.sqrt(rho))
    return CgResult(x, j, float(np.sqrt(rho)), bnorm, term, alphas, betas, rnorms)
