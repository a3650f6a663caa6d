"""Pins for oracle/cg.py (Algorithm 1 CG; Theorems 1-5)."""
import json
import os

import numpy as np
import pytest

from cs_inputs import draw_sign_bits, draw_rows, rng
from oracle import SrmOperator, DenseOperator, cg, reduced_cg, lstsq_on_support
from oracle.dense import columns

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _srm(N, M, seed):
    return SrmOperator(N, draw_sign_bits(N, rng(98, seed, N, 0)), draw_rows(N, M, rng(98, seed, N, 1)))


def test_cg_identity_worked_example():
    g = GOLD["cg_identity"]
    op = DenseOperator(np.eye(4))
    y = np.array(g["y"], float)
    S = np.array(g["S"])
    res = cg(op, S, op.adjoint(y), tol=1e-13)
    theta = np.zeros(4)
    theta[S] = res.x
    np.testing.assert_allclose(theta, g["theta"], atol=1e-14)
    assert res.iters <= g["max_iters"]


@pytest.mark.parametrize("seed", range(8))
def test_cg_equals_pseudo_inverse_ls(seed):
    """BASELINE.json oracle check (2): CG (Thm 1-2) == closed-form LS on small supports to 1e-10."""
    N, M = 4096, 1024      # |S| <= 256 = M/4, the well-posed regime of the configs
    op = _srm(N, M, seed)
    g = np.random.default_rng(seed)
    k = [1, 7, 32, 100, 160, 200, 230, 256][seed]
    S = np.sort(g.choice(N, k, replace=False))
    y = g.standard_normal(M)
    res = cg(op, S, op.adjoint(y), tol=1e-14)
    AS = columns(op, S)
    ref = np.linalg.pinv(AS) @ y
    assert np.linalg.norm(res.x - ref) <= 1e-10 * np.linalg.norm(ref)
    ref2 = lstsq_on_support(op, S, y)
    assert np.linalg.norm(ref2 - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("seed", range(5))
def test_residual_orthogonal_to_selected_columns(seed):
    """BASELINE.json oracle check (3): A_S^T (y - A_S x) ~ 0 after CG."""
    N, M = 4096, 1024
    op = _srm(N, M, seed)
    g = np.random.default_rng(100 + seed)
    S = np.sort(g.choice(N, 128, replace=False))
    y = g.standard_normal(M)
    c0 = op.adjoint(y)
    res = cg(op, S, c0, tol=1e-12)
    xt = np.zeros(N)
    xt[S] = res.x
    grad = op.adjoint(y - op.apply(xt))[S]
    assert np.linalg.norm(grad) <= 1e-11 * np.linalg.norm(c0[S])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_theorem4_k_distinct_eigenvalues(k):
    """Thm 4: H with k distinct eigenvalues -> CG ends in <= k iterations."""
    g = np.random.default_rng(k)
    M, N, s = 40, 60, 9
    for trial in range(10):
        Q, _ = np.linalg.qr(g.standard_normal((M, M)))
        norms = np.array([1.0, 2.5, 4.0][:k])[np.arange(s) % k]
        A = g.standard_normal((M, N))
        S = np.sort(g.choice(N, s, replace=False))
        A[:, S] = Q[:, :s] * norms          # orthogonal columns, k distinct norms
        op = DenseOperator(A)
        y = g.standard_normal(M)
        res = cg(op, S, op.adjoint(y), tol=1e-12)
        assert res.iters <= k, (trial, res.iters)


def test_theorem5_masked_iterates_equal_reduced_system():
    """Thm 5 proof: masked CG on Eq.(11) steps exactly as CG on Eq.(12)."""
    g = np.random.default_rng(5)
    for trial in range(20):
        M, N = 32, 64
        A = g.standard_normal((M, N))
        s = 1 + trial % 8
        S = np.sort(g.choice(N, s, replace=False))
        y = g.standard_normal(M)
        op = DenseOperator(A)
        full = cg(op, S, op.adjoint(y), tol=1e-13, trace=True)
        red = reduced_cg(A[:, S], y, tol=1e-13)
        assert full.iters == red.iters
        assert full.iters <= s + 2                      # S:482 acceptance 2
        np.testing.assert_allclose(full.alphas, red.alphas, rtol=1e-9)
        np.testing.assert_allclose(full.rnorms, red.rnorms, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(full.x, np.linalg.lstsq(A[:, S], y, rcond=None)[0], rtol=1e-8, atol=1e-10)


def test_warm_start_at_solution_takes_zero_iterations():
    N, M = 512, 128
    op = _srm(N, M, 1)
    g = np.random.default_rng(1)
    S = np.sort(g.choice(N, 20, replace=False))
    y = g.standard_normal(M)
    c0 = op.adjoint(y)
    x = cg(op, S, c0, tol=1e-14).x
    res = cg(op, S, c0, x0=x, tol=1e-10)
    assert res.iters == 0


def test_theorem3_zero_rhs_and_convergence():
    # b = 0 (y orthogonal to the selected columns): loop never runs, x stays 0.
    op = DenseOperator(np.eye(4))
    res = cg(op, np.array([0, 2]), op.adjoint(np.array([0.0, 1.0, 0.0, 1.0])))
    assert res.iters == 0 and not np.any(res.x)
