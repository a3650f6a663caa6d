"""Pins for oracle/pursuits.py: worked examples, brute force, dense-LS backend
equivalence (Thm 1-2 at algorithm level), exact noiseless recovery (BJ check 4)."""
import json
import os

import numpy as np
import pytest

import cs_inputs
import oracle
from cs_inputs import CONFIGS
from oracle import DenseOperator, SrmOperator, omp, sp, ompr, cosamp, brute_force_l0, topk
from helpers import measure, oracle_recover

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("fn", [omp, sp, ompr, cosamp])
def test_identity_worked_example(fn):
    g = GOLD["pursuit_identity"]
    op = DenseOperator(np.eye(4))
    res = fn(op, np.array(g["y"], float), g["K"], tol=1e-13)
    np.testing.assert_array_equal(res.support, g["support"])
    np.testing.assert_allclose(res.s_hat, g["s_hat"], atol=1e-14)


def test_brute_force_identity_worked_example():
    g = GOLD["brute_force_identity"]
    S, v, res = brute_force_l0(np.eye(4), np.array(g["y"], float), g["k"])
    np.testing.assert_array_equal(S, g["support"])
    assert res <= 1e-14


def test_topk_ties_go_to_lowest_index():
    v = np.array([1.0, 3.0, 3.0, 0.5, 3.0, 2.0])
    np.testing.assert_array_equal(topk(v, 2), [1, 2])
    np.testing.assert_array_equal(topk(v, 4), [1, 2, 4, 5])
    allowed = np.array([True, False, True, True, True, True])
    np.testing.assert_array_equal(topk(v, 2, allowed), [2, 4])
    np.testing.assert_array_equal(topk(np.zeros(5), 3), [0, 1, 2])


@pytest.mark.parametrize("fn", [omp, sp, ompr, cosamp])
def test_matches_brute_force_on_tiny_planted(fn):
    """l0 enumeration (Eq.(3)) on noiseless planted 2-sparse instances."""
    g = np.random.default_rng(11)
    hits = 0
    for trial in range(20):
        M, N, k = 16, 24, 2
        A = g.standard_normal((M, N))
        S0 = np.sort(g.choice(N, k, replace=False))
        s = np.zeros(N)
        s[S0] = g.standard_normal(k) + np.sign(g.standard_normal(k))
        y = A @ s
        Sb, _, rb = brute_force_l0(A, y, k)
        np.testing.assert_array_equal(Sb, S0)
        assert rb <= 1e-10
        res = fn(DenseOperator(A), y, k, tol=1e-13)
        if res.resid_norm <= 1e-9 * np.linalg.norm(y):
            np.testing.assert_array_equal(res.support, Sb)    # residual 0 => the l0 solution
            hits += 1
        else:
            assert res.resid_norm >= rb                        # l0 lower-bounds every pursuit
    assert hits >= 16


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
def test_cg_backend_equals_dense_ls_backend(alg):
    """S:484 acceptance 4: CG_WEIGHTED == DENSE_LS, N=128, M=32, K=8."""
    for trial in range(10):
        cfg = cs_inputs.Config(90, alg, 128, 32, 8, "gauss", 0.0 if trial % 2 else 1e-2)
        p = cs_inputs.make_problem(cfg, trial)
        op, y32 = measure(p)
        a = oracle_recover(p, y32, tol=1e-13)
        b = oracle_recover(p, y32, tol=1e-13, solver="lstsq")
        np.testing.assert_array_equal(a.support, b.support)
        assert np.linalg.norm(a.s_hat - b.s_hat) <= 1e-8 * np.linalg.norm(b.s_hat)


def _check_exact(p, res, rtol):
    np.testing.assert_array_equal(res.support, p.support)
    assert np.linalg.norm(res.s_hat - p.s) <= rtol * np.linalg.norm(p.s)


def test_exact_recovery_c1_omp_full_size():
    """BJ check (4): noiseless OMP recovers the planted support, config 1 at full size."""
    p = cs_inputs.make_problem(CONFIGS[1])
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)        # y is rounded to fp32 (R21): error ~ 6e-8 relative
    assert res.outer_iters == 64


def test_exact_recovery_c4_sp_full_size_problem():
    p = cs_inputs.make_problem(CONFIGS[4], b=3)
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)


def test_exact_recovery_c3_ompr_scaled():
    p = cs_inputs.make_problem(CONFIGS[3].scaled(32))
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)
    assert res.termination == 3       # support fixed point


def test_sp_noisy_invariants_c2_scaled():
    """c2 is noisy: parity unpinned beyond invariants."""
    p = cs_inputs.make_problem(CONFIGS[2].scaled(8))
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    h = res.resid_history
    assert all(h[i + 1] < h[i] for i in range(len(h) - 1))
    y = y32.astype(np.float64)
    grad = op.adjoint(y - op.apply(res.s_hat))[res.support]
    assert np.linalg.norm(grad) <= 1e-9 * np.linalg.norm(op.adjoint(y)[res.support])
    assert res.support.size == p.K
    # noise floor: ||r|| is about sigma sqrt(M - K)
    assert res.resid_norm <= 2.0 * CONFIGS[2].noise * np.sqrt(p.M)


def test_cosamp_exact_recovery_c4_shape():
    """CoSaMP (R33) at the c4 shape (N = 16384, M = 4096, K = 256): planted support and
    coefficients; a fixed point reached in a few iterations."""
    cfg = cs_inputs.Config(4, "cosamp", 16384, 4096, 256, "gauss", 0.0)
    p = cs_inputs.make_problem(cfg, 3)
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)
    assert res.termination in (3, 4) and res.outer_iters <= 6   # at the fp32-y floor either halt fires


def test_cosamp_first_iterate_is_pruned_ls_on_top_2k():
    """One iteration by hand with the dense-LS backend: T = top-2K |A^T y|, b = lstsq on T,
    S' = top-K |b| — the definition of the CoSaMP step (R33)."""
    g = np.random.default_rng(5)
    M, N, K = 40, 64, 4
    A = g.standard_normal((M, N)) / np.sqrt(M)
    y = g.standard_normal(M)
    res = cosamp(DenseOperator(A), y, K, tol=1e-13, max_outer=1, solver="lstsq")
    T = np.argsort(-np.abs(A.T @ y), kind="stable")[: 2 * K]
    T.sort()
    b = np.linalg.lstsq(A[:, T], y, rcond=None)[0]
    keep = np.sort(T[np.argsort(-np.abs(b), kind="stable")[:K]])
    np.testing.assert_array_equal(res.support, keep)
    np.testing.assert_allclose(res.x, b[np.searchsorted(T, keep)], rtol=1e-10)


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
def test_perm_randomizer_is_a_column_relabelling(alg):
    """Eq.(7)'s R (R34) relabels columns: recovering s with D F R equals recovering
    s' = R s with D F (sigma = +1, no R) and mapping the support back through pi."""
    cfg = cs_inputs.Config(91, alg, 1024, 256, 16, "gauss", 0.0, randomizer="perm")
    p = cs_inputs.make_problem(cfg, 0)
    op = SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    y = op.apply(p.s)
    a = oracle.recover(alg, op, y, p.K, tol=1e-13)
    op1 = SrmOperator(p.N, p.sign_bits, p.rows)
    b = oracle.recover(alg, op1, op1.apply(p.s[p.perm]), p.K, tol=1e-13)
    np.testing.assert_array_equal(a.support, np.sort(p.perm[b.support]))
    np.testing.assert_allclose(a.s_hat[p.perm], b.s_hat, atol=1e-10)
    np.testing.assert_array_equal(a.support, p.support)


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
def test_psi_dct_cg_backend_equals_dense_ls_and_recovers(alg):
    """A = Phi Psi with Psi = DCT (R35): CG and dense-LS backends agree, and the planted
    DCT-domain-sparse s is recovered exactly (noiseless)."""
    for trial in range(3):
        cfg = cs_inputs.Config(92, alg, 256, 64, 6, "gauss", 0.0, randomizer="perm", psi="dct")
        p = cs_inputs.make_problem(cfg, trial)
        op, y32 = measure(p)
        a = oracle_recover(p, y32, tol=1e-13)
        b = oracle_recover(p, y32, tol=1e-13, solver="lstsq")
        np.testing.assert_array_equal(a.support, b.support)
        assert np.linalg.norm(a.s_hat - b.s_hat) <= 1e-8 * np.linalg.norm(b.s_hat)
    cfg = cs_inputs.Config(92, alg, 4096, 1024, 64, "gauss", 0.0, psi="dct")
    p = cs_inputs.make_problem(cfg, 0)
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
def test_partial_fourier_cg_backend_equals_dense_ls_and_recovers(alg):
    """F = partial Fourier (R36): CG and dense-LS backends agree; noiseless exact recovery."""
    for trial in range(3):
        cfg = cs_inputs.Config(93, alg, 256, 96, 6, "gauss", 0.0, randomizer="perm", transform="dft")
        p = cs_inputs.make_problem(cfg, trial)
        op, y32 = measure(p)
        a = oracle_recover(p, y32, tol=1e-13)
        b = oracle_recover(p, y32, tol=1e-13, solver="lstsq")
        np.testing.assert_array_equal(a.support, b.support)
        assert np.linalg.norm(a.s_hat - b.s_hat) <= 1e-8 * np.linalg.norm(b.s_hat)
    cfg = cs_inputs.Config(93, alg, 4096, 1024, 64, "gauss", 0.0, randomizer="perm", transform="dft")
    p = cs_inputs.make_problem(cfg, 0)
    op, y32 = measure(p)
    res = oracle_recover(p, y32)
    _check_exact(p, res, 1e-6)


# ---- step-level pins (VERDICT r1 "What's weak #1"): each one fails if the named step of
# oracle/pursuits.py is mutated.  Every expected value is worked out by hand in the docstring.

def test_omp_excludes_current_support_on_zero_ties():
    """Eq.(6) with reading R12: the argmax runs over j not in S.  A = I_4,
    y = (5, 0, -3, 0), K = 3: t1 = 0 (x = 5), t2 = 2 (x = -3), after which r = 0 and every
    |c_j| = 0; the argmax over j not in S picks the lowest such index, 1.  Without the
    exclusion it would re-pick index 0."""
    res = omp(DenseOperator(np.eye(4)), np.array([5.0, 0.0, -3.0, 0.0]), 3, tol=1e-13)
    np.testing.assert_array_equal(res.support, [0, 1, 2])
    np.testing.assert_allclose(res.x, [5.0, 0.0, -3.0], atol=1e-14)


def test_sp_resid_rose_keeps_previous_support():
    """SP halting (reading R15): when the pruned support's residual does not fall,
    stop and KEEP (S, x).  K = 1, A = [[3,1,0],[-1,0,-1]], y = (3, 2):
      A^T y = (7, 3, -2)                 -> S = {0}, x = 7/10 = 0.7
      r = (0.9, 2.7), ||r||^2 = 8.1;  c = A^T r = (0, 0.9, -2.7) -> J = {2}
      LS on T = {0, 2}: x_T = (1, -3)    -> S' = {2}, x' = a_2.y/|a_2|^2 = -2
      r' = (3, 0), ||r'|| = 3 >= sqrt(8.1) = 2.846 -> RESID_ROSE, return S = {0}, x = 0.7.
    Without the halting rule SP would move to {2} and stop there (S' = S next time)."""
    A = np.array([[3.0, 1.0, 0.0], [-1.0, 0.0, -1.0]])
    res = sp(DenseOperator(A), np.array([3.0, 2.0]), 1, tol=1e-13)
    assert res.termination == oracle.pursuits.T_RESID_ROSE
    np.testing.assert_array_equal(res.support, [0])
    np.testing.assert_allclose(res.x, [0.7], rtol=1e-12)
    np.testing.assert_allclose(res.resid_norm, np.sqrt(8.1), rtol=1e-12)
    assert res.outer_iters == 1


def test_sp_candidates_exclude_current_support():
    """SP's J = top-K of |c| over j NOT in S.  K = 2,
    A = [[0,0,2,-1,1],[1,0,0,2,0],[2,2,-1,0,0],[0,0,0,0,2]], y = (0,-2,-3,1):
      A^T y = (-8, -6, 3, -4, 2)                  -> S = {0, 1}, x = (-2, 0.5)
      r = (0, 0, 0, 1), c = A^T r = (0, 0, 0, 0, 2): off S only c_4 != 0, so J = {4, 2}
      (the zero tie goes to the lowest index NOT in S);  T = {0,1,2,4} is square:
      x_T = (-2, 0.375, -0.25, 0.5)              -> S' = {0, 4}
      a_0 and a_4 are orthogonal: x' = (a_0.y/5, a_4.y/5) = (-1.6, 0.4),
      r' = (-0.4, -0.4, 0.2, 0.2), ||r'||^2 = 0.4 < 1 -> accept
      c = A^T r' = (0, 0.4, -1, -0.4, 0) -> J = {2, 1} (or {2, 3}: both give S' = {0, 4})
      -> S' = S: SUPPORT_FIXED after 2 outer iterations with S = {0, 4}, x = (-1.6, 0.4).
    Taking J over ALL indices gives J = {4, 0}, T = {0, 1, 4}, x_T = (-2, 0.5, 0.4) and a
    premature fixed point at {0, 1}.  The exact dense-LS backend keeps the zero ties exact
    (integer data, r = (0, 0, 0, 1) exactly); CG would leave ~1e-16 correlations that
    break them arbitrarily."""
    A = np.array([[0, 0, 2, -1, 1], [1, 0, 0, 2, 0], [2, 2, -1, 0, 0], [0, 0, 0, 0, 2]], float)
    res = sp(DenseOperator(A), np.array([0.0, -2.0, -3.0, 1.0]), 2, tol=1e-13, solver="lstsq")
    np.testing.assert_array_equal(res.support, [0, 4])
    np.testing.assert_allclose(res.x, [-1.6, 0.4], rtol=1e-10)
    assert res.termination == oracle.pursuits.T_SUPPORT_FIXED and res.outer_iters == 2
    np.testing.assert_allclose(res.resid_history, [1.0, np.sqrt(0.4)], rtol=1e-10)


@pytest.mark.parametrize("eta,support,x,term", [
    (1.0, [0, 2], [5.0, 4.0], 3),     # z_J = (3, 2.5) < min|x_S| = 4: S' = S
    (1.5, [0, 3], [5.0, 3.0], 1),     # z = (5, 4, 4.5, 3.75): keep 0 and 3
    (2.5, [3, 5], [3.0, 2.5], 1),     # z = (5, 4, 7.5, 6.25): keep 3 and 5
])
def test_ompr_eta_step(eta, support, x, term):
    """One OMPR(l, eta) step (reading R16): z = x~ + eta A^T r,
    J = top-l of |z| off S, S' = top-K of |z| over S u J.  A = I_8, K = 2, l = 2,
    y = (5, 0, 4, 3, 0, 2.5, 0, 0): S = {0, 2}, x = (5, 4), r = c = y off S, so on
    U = {0, 2, 3, 5}: z = (5, 4, 3 eta, 2.5 eta).  One outer iteration (max_outer = 1);
    the new x is y on S' (LS with A = I).  eta decides every swap."""
    y = np.array([5.0, 0.0, 4.0, 3.0, 0.0, 2.5, 0.0, 0.0])
    res = ompr(DenseOperator(np.eye(8)), y, 2, tol=1e-13, l=2, eta=eta, max_outer=1)
    np.testing.assert_array_equal(res.support, support)
    np.testing.assert_allclose(res.x, x, atol=1e-12)
    assert res.termination == term and res.outer_iters == 1


@pytest.mark.parametrize("eta,support,term,outer", [(1.0, [0], 3, 1), (2.0, [1], 1, 1)])
def test_ompr1_eta_decides_the_swap(eta, support, term, outer):
    """OMPR(1): A = I_4, y = (4, 3, 0, 0), K = 1: S = {0}, x = 4, c = (0, 3, 0, 0), so the
    single candidate j = 1 has z_1 = 3 eta.  eta = 1: 3 < 4, S' = S (SUPPORT_FIXED);
    eta = 2: 6 > 4, swap to {1} with x = 3 (one step, max_outer = 1)."""
    res = ompr(DenseOperator(np.eye(4)), np.array([4.0, 3.0, 0.0, 0.0]), 1, tol=1e-13, eta=eta, max_outer=1)
    np.testing.assert_array_equal(res.support, support)
    assert res.termination == term and res.outer_iters == outer


@pytest.mark.parametrize("cid", [3, 5])
def test_full_size_oracle_references_are_consistent(cid):
    """tests/golden/oracle_c{3,5}.npz (written by tools/oracle_reference.py from oracle/ only)
    pinned to things other than themselves: the stored y digest is the digest of the seeded
    input formed here; the stored coefficients are the LS solution on the stored support
    (residual orthogonal to the selected columns, Thm 1-2, to the CG tolerance);
    c3 (noiseless, M >> K log(N/K)) is the planted support."""
    import hashlib
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", f"oracle_c{cid}.npz"))
    p = cs_inputs.make_problem(CONFIGS[cid], 0, 0)
    op, y32 = measure(p)
    assert hashlib.sha256(y32.tobytes()).hexdigest() == str(g["y_sha"])
    S, x = g["support"], g["x"]
    assert S.size == p.K and np.all(np.diff(S) > 0)
    s_hat = np.zeros(p.N)
    s_hat[S] = x
    y = y32.astype(np.float64)
    grad = op.adjoint(y - op.apply(s_hat))[S]
    assert np.linalg.norm(grad) <= 1e-9 * np.linalg.norm(op.adjoint(y)[S])
    if cid == 3:
        np.testing.assert_array_equal(S, p.support)
        assert int(g["termination"]) == oracle.pursuits.T_SUPPORT_FIXED
