"""Dense small-scale references (fp64).  TEST INFRASTRUCTURE.

* lstsq_on_support — the plain definition the CG step must reach:
  s_S = argmin ||y - A_S v||_2 (Eq.(9); Theorems 1-2),
  via numpy.linalg.lstsq on the materialised columns A_S (tiny N only).
* brute_force_l0 — Eq.(3) by enumeration of all k-subsets
  (S:365-373); oracle for tiny instances only.
"""
from __future__ import annotations

import itertools

import numpy as np


def columns(op, S):
    """A_S materialised column by column via A e_j."""
    S = np.asarray(S, dtype=np.int64)
    cols = []
    for j in S:
        e = np.zeros(op.N)
        e[j] = 1.0
        cols.append(op.apply(e))
    return np.stack(cols, axis=1) if cols else np.zeros((op.M, 0))


def lstsq_on_support(op, S, y):
    AS = columns(op, S)
    return np.linalg.lstsq(AS, np.asarray(y, dtype=np.float64), rcond=None)[0]


def brute_force_l0(A: np.ndarray, y: np.ndarray, k: int):
    """Minimal-residual k-subset (ties: lexicographically first).  N <= 24, k <= 4."""
    M, N = A.shape
    if N > 24 or k > 4:
        raise ValueError("brute force guard: N <= 24, k <= 4")
    if k == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0), float(np.linalg.norm(y))
    best = None
    for S in itertools.combinations(range(N), k):
        AS = A[:, S]
        v = np.linalg.lstsq(AS, y, rcond=None)[0]
        res = float(np.linalg.norm(y - AS @ v))
        if best is None or res < best[2] - 1e-12:
            best = (np.array(S, dtype=np.int64), v, res)
    return best
