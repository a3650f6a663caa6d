"""Pins for oracle/operator.py against facts fixed by the paper and the mathematics.

The oracle applies A with scipy's DCT; these tests check it against (a) the
explicit DCT-II definition written as a matrix, (b) closed-form DCT
facts (constant and cosine inputs), (c) SPEC's worked examples, and (d) the
structural invariants A A^T = I_M, adjoint identity, linearity.
"""
import json
import os

import numpy as np
import pytest
import scipy.fft

from cs_inputs import pack_sign_bits, draw_sign_bits, draw_rows, draw_perm, rng
from oracle import SrmOperator, dct_matrix, dense_srm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _op(N, M, seed=0):
    bits = draw_sign_bits(max(N, 32), rng(99, seed, N, 0))
    rows = draw_rows(N, M, rng(99, seed, N, 1))
    return SrmOperator(N, bits, rows), bits, rows


def test_dct_constant_worked_example():
    g = GOLD["dct_constant"]
    op = SrmOperator(4, pack_sign_bits(np.zeros(4, bool)), np.arange(4))
    np.testing.assert_allclose(op.apply(np.array(g["x"], float)), g["X"], atol=1e-15)
    gi = GOLD["dct_inverse_constant"]
    np.testing.assert_allclose(op.adjoint(np.array(gi["X"], float)), gi["x"], atol=1e-15)


@pytest.mark.parametrize("N", [4, 8, 32, 256])
def test_dct_cosine_inputs_are_impulses(N):
    # u_n = cos(pi (2n+1) k0 / 2N) is row k0 of the unnormalised DCT-II basis;
    # with orthonormal scaling X = sqrt(N/2) e_k0 (k0 >= 1), sqrt(N) e_0 for k0 = 0.
    op = SrmOperator(N, pack_sign_bits(np.zeros(N, bool)), np.arange(N))
    n = np.arange(N)
    for k0 in [0, 1, N // 2, N - 1]:
        u = np.cos(np.pi * (2 * n + 1) * k0 / (2 * N))
        X = op.apply(u)
        e = np.zeros(N)
        e[k0] = np.sqrt(N) if k0 == 0 else np.sqrt(N / 2)
        np.testing.assert_allclose(X, e, atol=1e-12 * np.sqrt(N))


@pytest.mark.parametrize("N,M", [(8, 2), (16, 4), (64, 16), (256, 64), (1024, 256), (4096, 1024)])
def test_operator_matches_dense_definition(N, M):
    """BASELINE.json oracle check (1): operator and adjoint exact to 1e-12 vs explicit A."""
    op, bits, rows = _op(N, M)
    A = dense_srm(N, bits, rows)
    g = np.random.default_rng(N)
    for _ in range(3):
        x = g.standard_normal(N)
        w = g.standard_normal(M)
        np.testing.assert_allclose(op.apply(x), A @ x, atol=1e-12 * np.linalg.norm(x))
        np.testing.assert_allclose(op.adjoint(w), A.T @ w, atol=1e-12 * np.linalg.norm(w))


def test_dct_matrix_is_orthonormal():
    for N in [4, 16, 128]:
        C = dct_matrix(N)
        np.testing.assert_allclose(C @ C.T, np.eye(N), atol=1e-13)
    # and equals scipy's orthonormal DCT-II applied to the identity (independent routine)
    C = dct_matrix(64)
    np.testing.assert_allclose(C, scipy.fft.dct(np.eye(64), type=2, norm="ortho", axis=0), atol=1e-13)


@pytest.mark.parametrize("N,M", [(32, 8), (256, 64), (2048, 512)])
def test_rows_orthonormal_AAT_identity(N, M):
    """unscaled SRM with orthonormal transform has A A^T = I_M."""
    op, _, _ = _op(N, M)
    AAT = np.stack([op.apply(op.adjoint(e)) for e in np.eye(M)], axis=1)
    np.testing.assert_allclose(AAT, np.eye(M), atol=1e-13)


def test_adjoint_identity_linearity_zero():
    N, M = 1 << 14, 1 << 12
    op, _, _ = _op(N, M, seed=3)
    g = np.random.default_rng(7)
    for _ in range(10):
        x, w = g.standard_normal(N), g.standard_normal(M)
        lhs, rhs = op.apply(x) @ w, x @ op.adjoint(w)
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(w)
    x, z = g.standard_normal(N), g.standard_normal(N)
    np.testing.assert_allclose(op.apply(2 * x - 3 * z), 2 * op.apply(x) - 3 * op.apply(z), atol=1e-11)
    assert not np.any(op.apply(np.zeros(N)))
    assert not np.any(op.adjoint(np.zeros(M)))


def test_sign_diagonal_effect():
    # flipping sigma_j flips column j of A exactly
    N, M = 64, 16
    bits0 = pack_sign_bits(np.zeros(N, bool))
    neg = np.zeros(N, bool)
    neg[5] = True
    bits1 = pack_sign_bits(neg)
    rows = np.arange(0, N, 4)
    A0, A1 = dense_srm(N, bits0, rows), dense_srm(N, bits1, rows)
    np.testing.assert_array_equal(A1[:, 5], -A0[:, 5])
    np.testing.assert_array_equal(np.delete(A1, 5, 1), np.delete(A0, 5, 1))


def test_first_row_is_mean_scaled():
    # C_N[0, :] = 1/sqrt(N): with rows = [0] and sigma = +1, A x = sum(x)/sqrt(N)
    N = 32
    op = SrmOperator(N, pack_sign_bits(np.zeros(N, bool)), np.array([0]))
    x = np.arange(N, dtype=float)
    np.testing.assert_allclose(op.apply(x), [x.sum() / np.sqrt(N)], rtol=1e-14)


# ---------------------------------------------------------------- Eq.(7) randomizer R = pi (R34)
@pytest.mark.parametrize("N,M", [(8, 2), (64, 16), (512, 128)])
def test_perm_operator_matches_dense_definition(N, M):
    """A = C_N[rows] R diag(sigma) with R the explicit permutation matrix R[i, pi(i)] = 1."""
    bits = draw_sign_bits(max(N, 32), rng(97, 0, N, 0))
    rows = draw_rows(N, M, rng(97, 0, N, 1))
    perm = draw_perm(N, rng(97, 0, N, 2))
    op = SrmOperator(N, bits, rows, perm)
    A = dense_srm(N, bits, rows, perm)
    g = np.random.default_rng(N + 1)
    for _ in range(3):
        x, w = g.standard_normal(N), g.standard_normal(M)
        np.testing.assert_allclose(op.apply(x), A @ x, atol=1e-12 * np.linalg.norm(x))
        np.testing.assert_allclose(op.adjoint(w), A.T @ w, atol=1e-12 * np.linalg.norm(w))


def test_perm_columns_are_permuted_dct_columns():
    """Column j of D F R is column pi^{-1}(j) of the row-sampled DCT (the randomizer only
    relabels columns, Eq.(7)): A e_j = C_N[rows, pi^{-1}(j)]."""
    N, M = 128, 32
    perm = draw_perm(N, rng(97, 1, N, 2))
    pinv = np.argsort(perm)
    rows = draw_rows(N, M, rng(97, 1, N, 1))
    op = SrmOperator(N, pack_sign_bits(np.zeros(N, bool)), rows, perm)
    C = dct_matrix(N)
    for j in [0, 1, 5, 77, N - 1]:
        e = np.zeros(N)
        e[j] = 1.0
        np.testing.assert_allclose(op.apply(e), C[rows, pinv[j]], atol=1e-14)


def test_perm_operator_rows_orthonormal_and_adjoint():
    N, M = 2048, 512
    perm = draw_perm(N, rng(97, 2, N, 2))
    op = SrmOperator(N, draw_sign_bits(N, rng(97, 2, N, 0)), draw_rows(N, M, rng(97, 2, N, 1)), perm)
    AAT = np.stack([op.apply(op.adjoint(e)) for e in np.eye(M)[:64]], axis=1)
    np.testing.assert_allclose(AAT, np.eye(M)[:, :64], atol=1e-13)
    g = np.random.default_rng(3)
    x, w = g.standard_normal(N), g.standard_normal(M)
    assert abs(op.apply(x) @ w - x @ op.adjoint(w)) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(w)


# ---------------------------------------------------------------- Psi = DCT (A = Phi Psi, R35)
@pytest.mark.parametrize("N,M,use_perm", [(16, 4, False), (64, 16, True), (512, 128, True)])
def test_psi_dct_operator_matches_dense_definition(N, M, use_perm):
    """A = C_N[rows] R diag(sigma) C_N with explicit cosine matrices on the dense side."""
    bits = draw_sign_bits(max(N, 32), rng(96, 0, N, 0))
    rows = draw_rows(N, M, rng(96, 0, N, 1))
    perm = draw_perm(N, rng(96, 0, N, 2)) if use_perm else None
    op = SrmOperator(N, bits, rows, perm, psi="dct")
    A = dense_srm(N, bits, rows, perm, psi="dct")
    g = np.random.default_rng(N + 2)
    for _ in range(3):
        x, w = g.standard_normal(N), g.standard_normal(M)
        np.testing.assert_allclose(op.apply(x), A @ x, atol=1e-12 * np.linalg.norm(x))
        np.testing.assert_allclose(op.adjoint(w), A.T @ w, atol=1e-12 * np.linalg.norm(w))


def test_psi_dct_columns_are_phi_of_dct_basis_vectors():
    """x = Psi s: column j of A = Phi Psi is Phi applied to column j of C_N."""
    N, M = 128, 32
    bits = draw_sign_bits(N, rng(96, 1, N, 0))
    rows = draw_rows(N, M, rng(96, 1, N, 1))
    phi = SrmOperator(N, bits, rows)
    A = SrmOperator(N, bits, rows, psi="dct")
    C = dct_matrix(N)
    for j in [0, 3, 64, N - 1]:
        e = np.zeros(N)
        e[j] = 1.0
        np.testing.assert_allclose(A.apply(e), phi.apply(C[:, j]), atol=1e-13)


def test_psi_dct_rows_orthonormal():
    N, M = 1024, 256
    op = SrmOperator(N, draw_sign_bits(N, rng(96, 2, N, 0)), draw_rows(N, M, rng(96, 2, N, 1)),
                     draw_perm(N, rng(96, 2, N, 2)), psi="dct")
    AAT = np.stack([op.apply(op.adjoint(e)) for e in np.eye(M)[:48]], axis=1)
    np.testing.assert_allclose(AAT, np.eye(M)[:, :48], atol=1e-13)


# ---------------------------------------------------------------- F = partial Fourier (R36)
from cs_inputs import draw_freqs  # noqa: E402
from oracle.operator import dft_rows_matrix  # noqa: E402


@pytest.mark.parametrize("N,Mf,use_perm", [(8, 2, False), (64, 12, True), (1024, 200, True)])
def test_dft_operator_matches_dense_definition(N, Mf, use_perm):
    """Explicit cos / sin rows (no FFT) against the FFT-based oracle operator."""
    bits = draw_sign_bits(max(N, 32), rng(95, 0, N, 0))
    freqs = draw_freqs(N, Mf, rng(95, 0, N, 1))
    perm = draw_perm(N, rng(95, 0, N, 2)) if use_perm else None
    op = SrmOperator(N, bits, freqs, perm, transform="dft")
    A = dense_srm(N, bits, freqs, perm, transform="dft")
    assert A.shape == (2 * Mf, N) and op.M == 2 * Mf
    g = np.random.default_rng(N + 3)
    for _ in range(3):
        x, w = g.standard_normal(N), g.standard_normal(2 * Mf)
        np.testing.assert_allclose(op.apply(x), A @ x, atol=1e-12 * np.linalg.norm(x))
        np.testing.assert_allclose(op.adjoint(w), A.T @ w, atol=1e-12 * np.linalg.norm(w))


def test_dft_worked_example_cosine_input():
    """x_n = cos(2 pi f0 n / N) gives X_f0 = N/2 (real) and nothing at other frequencies:
    y = sqrt(2/N) (N/2, 0) at f0 = sqrt(N/2) (1, 0)."""
    N = 64
    f0 = 5
    x = np.cos(2 * np.pi * f0 * np.arange(N) / N)
    op = SrmOperator(N, pack_sign_bits(np.zeros(N, bool)), np.array([3, f0, 17]), transform="dft")
    np.testing.assert_allclose(op.apply(x), [0, 0, np.sqrt(N / 2), 0, 0, 0], atol=1e-12)


def test_dft_rows_orthonormal():
    N, Mf = 2048, 300
    op = SrmOperator(N, draw_sign_bits(N, rng(95, 1, N, 0)), draw_freqs(N, Mf, rng(95, 1, N, 1)),
                     draw_perm(N, rng(95, 1, N, 2)), transform="dft")
    AAT = np.stack([op.apply(op.adjoint(e)) for e in np.eye(2 * Mf)[:64]], axis=1)
    np.testing.assert_allclose(AAT, np.eye(2 * Mf)[:, :64], atol=1e-13)
    C = dft_rows_matrix(16, [1, 7])
    np.testing.assert_allclose(C @ C.T, np.eye(4), atol=1e-14)
