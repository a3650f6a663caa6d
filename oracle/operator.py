"""Oracle sensing operator A = P . F . diag(sigma)  (fp64, CPU).  TEST INFRASTRUCTURE.

Paper: Eq.(7) Phi = D F R: D samples M of N rows
("randomly choose M indices"), F is an orthonormal DCT (P:309-313,
"DCT can be speeded by FFT"), R is a randomizer.  BASELINE.json
binds the randomizer to a +-1 sign diagonal and Psi = I (reading R1),
so A x = (C_N (sigma . x))[rows] and A^T w = sigma . C_N^T scatter_rows(w)
(SURVEY §8c.1).  The literal Eq.(7) randomizer R — a permutation pi,
(R u)_i = u_{pi(i)} — is the optional `perm` (reading R34):
A = P C_N R diag(sigma), with sigma = +1 for the paper's own D F R.  The
dictionary Psi of A = Phi Psi (x = Psi s) is I (BASELINE) or, with
`psi="dct"`, the orthonormal DCT-II C_N of the paper's experiments ("Psi is
chosen to be a discrete cosine transform"; reading R35).  C_N is the orthonormal DCT-II
    C_N[k, n] = c_k sqrt(2/N) cos(pi (2n+1) k / (2N)),  c_0 = 1/sqrt 2, else 1
(S:129), applied here with scipy.fft.dct(type=2, norm="ortho") and its
inverse; `dct_matrix` writes the same definition out as an explicit matrix for
tiny N (the check path, SURVEY §8c.1 "For N <= 4096, use a dense C_N").
"""
from __future__ import annotations

import numpy as np
import scipy.fft

from cs_inputs import unpack_sign_bits


def dct_matrix(N: int) -> np.ndarray:
    """Explicit orthonormal DCT-II matrix C_N, O(N^2): tiny N only."""
    k = np.arange(N)[:, None].astype(np.float64)
    n = np.arange(N)[None, :].astype(np.float64)
    C = np.sqrt(2.0 / N) * np.cos(np.pi * (2.0 * n + 1.0) * k / (2.0 * N))
    C[0, :] *= 1.0 / np.sqrt(2.0)
    return C


def dense_srm(N: int, sign_bits: np.ndarray, rows: np.ndarray, perm=None, psi=None) -> np.ndarray:
    """A = C_N[rows] R diag(sigma) Psi as a dense M x N matrix (tiny N only); R = I without
    `perm`, else the permutation matrix R[i, pi(i)] = 1; Psi = I, or C_N for psi="dct"."""
    sigma = np.where(unpack_sign_bits(sign_bits, N), -1.0, 1.0)
    R = np.eye(N)
    if perm is not None:
        R = np.zeros((N, N))
        R[np.arange(N), np.asarray(perm)] = 1.0
    A = (dct_matrix(N)[np.asarray(rows)] @ R) * sigma[None, :]
    if psi == "dct":
        A = A @ dct_matrix(N)
    return A


class SrmOperator:
    """Matrix-free A and A^T: O(N log N) time, O(N) memory."""

    def __init__(self, N: int, sign_bits: np.ndarray, rows: np.ndarray, perm=None, psi=None):
        self.N = int(N)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.M = self.rows.size
        self.sigma = np.where(unpack_sign_bits(sign_bits, N), -1.0, 1.0)
        self.perm = None if perm is None else np.asarray(perm, dtype=np.int64)
        assert psi in (None, "dct")
        self.psi = psi

    def apply(self, x: np.ndarray) -> np.ndarray:
        """A x = P C_N R (sigma . Psi x): Psi (DCT-II, ortho, for psi="dct"), sign, permute
        (u_i <- u_{pi(i)}), DCT-II (ortho), keep rows."""
        x = np.asarray(x, dtype=np.float64)
        if self.psi == "dct":
            x = scipy.fft.dct(x, type=2, norm="ortho")
        u = self.sigma * x
        if self.perm is not None:
            u = u[self.perm]
        X = scipy.fft.dct(u, type=2, norm="ortho")
        return X[self.rows]

    def adjoint(self, w: np.ndarray) -> np.ndarray:
        """A^T w = Psi^T sigma . R^T C_N^T P^T w: zero-fill unselected rows,
        DCT-III, un-permute (u_{pi(i)} <- v_i), sign, then Psi^T (DCT-III) for psi="dct"."""
        z = np.zeros(self.N)
        z[self.rows] = np.asarray(w, dtype=np.float64)
        v = scipy.fft.idct(z, type=2, norm="ortho")
        if self.perm is not None:
            u = np.zeros(self.N)
            u[self.perm] = v
            v = u
        v = self.sigma * v
        if self.psi == "dct":
            v = scipy.fft.idct(v, type=2, norm="ortho")      # Psi^T = C_N^T
        return v


class DenseOperator:
    """A given as an explicit matrix (M-OMP style); used for toy pins."""

    def __init__(self, A: np.ndarray):
        self.A = np.asarray(A, dtype=np.float64)
        self.M, self.N = self.A.shape

    def apply(self, x):
        return self.A @ np.asarray(x, dtype=np.float64)

    def adjoint(self, w):
        return self.A.T @ np.asarray(w, dtype=np.float64)
