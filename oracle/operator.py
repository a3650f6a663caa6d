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
chosen to be a discrete cosine transform"; reading R35).  With
`transform="dft"` F is the partial Fourier transform of the MRI case ("partial
Fourier transform is selected as the component F of ... DFR"; P:150,
P:263; reading R36): `rows` are frequencies f in [1, N/2 - 1] and each gives two
real measurements sqrt(2/N) (Re X_f, Im X_f), X = unnormalised DFT of R sigma x,
interleaved (y[2r], y[2r+1]) — the complex D F R y of a real signal, stacked and
scaled so the rows stay orthonormal.  C_N is the orthonormal DCT-II
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


def dft_rows_matrix(N: int, freqs) -> np.ndarray:
    """Explicit real partial-Fourier rows (R36): for each f, sqrt(2/N) cos(2 pi f n / N) and
    -sqrt(2/N) sin(2 pi f n / N) (real and imaginary part of e^{-2 pi i f n / N})."""
    n = np.arange(N, dtype=np.float64)[None, :]
    f = np.asarray(freqs, dtype=np.float64)[:, None]
    th = 2.0 * np.pi * f * n / N
    out = np.empty((2 * f.shape[0], N))
    out[0::2] = np.sqrt(2.0 / N) * np.cos(th)
    out[1::2] = -np.sqrt(2.0 / N) * np.sin(th)
    return out


def dense_srm(N: int, sign_bits: np.ndarray, rows: np.ndarray, perm=None, psi=None,
              transform="dct") -> np.ndarray:
    """A = C_N[rows] R diag(sigma) Psi as a dense M x N matrix (tiny N only); R = I without
    `perm`, else the permutation matrix R[i, pi(i)] = 1; Psi = I, or C_N for psi="dct"."""
    sigma = np.where(unpack_sign_bits(sign_bits, N), -1.0, 1.0)
    R = np.eye(N)
    if perm is not None:
        R = np.zeros((N, N))
        R[np.arange(N), np.asarray(perm)] = 1.0
    F = dct_matrix(N)[np.asarray(rows)] if transform == "dct" else dft_rows_matrix(N, rows)
    A = (F @ R) * sigma[None, :]
    if psi == "dct":
        A = A @ dct_matrix(N)
    return A


class SrmOperator:
    """Matrix-free A and A^T: O(N log N) time, O(N) memory."""

    def __init__(self, N: int, sign_bits: np.ndarray, rows: np.ndarray, perm=None, psi=None,
                 transform="dct"):
        self.N = int(N)
        self.rows = np.asarray(rows, dtype=np.int64)
        assert transform in ("dct", "dft")
        self.transform = transform
        self.M = self.rows.size * (2 if transform == "dft" else 1)
        self.sigma = np.where(unpack_sign_bits(sign_bits, N), -1.0, 1.0)
        self.perm = None if perm is None else np.asarray(perm, dtype=np.int64)
        assert psi in (None, "dct")
        self.psi = psi

    def apply(self, x: np.ndarray) -> np.ndarray:
        """A x = P F R (sigma . Psi x): Psi (DCT-II, ortho, for psi="dct"), sign, permute
        (u_i <- u_{pi(i)}), F = DCT-II (ortho) and keep rows, or F = DFT and keep
        sqrt(2/N) (Re, Im) of the selected frequencies (transform="dft", R36)."""
        x = np.asarray(x, dtype=np.float64)
        if self.psi == "dct":
            x = scipy.fft.dct(x, type=2, norm="ortho")
        u = self.sigma * x
        if self.perm is not None:
            u = u[self.perm]
        if self.transform == "dft":
            X = np.fft.fft(u)[self.rows] * np.sqrt(2.0 / self.N)
            y = np.empty(self.M)
            y[0::2], y[1::2] = X.real, X.imag
            return y
        X = scipy.fft.dct(u, type=2, norm="ortho")
        return X[self.rows]

    def adjoint(self, w: np.ndarray) -> np.ndarray:
        """A^T w = Psi^T sigma . R^T F^T P^T w: zero-fill unselected rows,
        DCT-III (or the real part of the inverse DFT of the selected frequencies, cf. P:263's
        IFFT([y;0])), un-permute (u_{pi(i)} <- v_i), sign, then Psi^T for psi="dct"."""
        w = np.asarray(w, dtype=np.float64)
        if self.transform == "dft":
            # x_n = sqrt(2/N) Re sum_f (w_re + i w_im)_f e^{+2 pi i f n / N}
            V = np.zeros(self.N, dtype=np.complex128)
            V[self.rows] = w[0::2] + 1j * w[1::2]
            v = np.sqrt(2.0 / self.N) * (self.N * np.fft.ifft(V)).real
        else:
            z = np.zeros(self.N)
            z[self.rows] = w
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
