"""The paper's literal Eq.(7) operator Phi = D F R with the permutation randomizer R
(R34) on the CUDA path, through the C ABI
(cs_operator_create_perm): operator and adjoint against the fp64 oracle on both tiers,
the device-side permutation check, and recovery parity (OMP, SP, OMPR, CoSaMP) including
the all-ties case, where selection must break ties by the ORIGINAL index."""
import ctypes

import numpy as np
import pytest

import cs_inputs
import oracle
from gpu_helpers import to_dev, perms_dev, measured, oracle_results, compare

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _probs(N, M, K, batch, alg="sp", seed=0, signal="gauss", noise=0.0):
    cfg = cs_inputs.Config(80 + seed, alg, N, M, K, signal, noise, randomizer="perm")
    return cfg, [cs_inputs.make_problem(cfg, b=b) for b in range(batch)]


def _op(cs, probs, dev, signs=False):
    bits, rows = to_dev(probs, dev)
    return cs.Operator(probs[0].N, probs[0].M, bits if signs else None, rows, batch=len(probs),
                       perm=perms_dev(probs, dev))


@pytest.mark.parametrize("N,M,batch", [(8, 4, 2), (64, 16, 3), (1024, 256, 2), (16384, 4096, 3),
                                       (32768, 8192, 1), (1 << 18, 1 << 16, 1)])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_perm_apply_adjoint_match_oracle(cs, N, M, batch, dtype):
    dev = torch.device("cuda:0")
    _, probs = _probs(N, M, max(1, M // 8), batch)
    A = _op(cs, probs, dev)
    g = np.random.default_rng(N)
    X, W = g.standard_normal((batch, N)), g.standard_normal((batch, M))
    td = getattr(torch, dtype)
    Yg = cs.cs_operator_apply(A, torch.from_numpy(X).to(dev, td)).cpu().numpy().astype(np.float64)
    Xg = cs.cs_operator_adjoint(A, torch.from_numpy(W).to(dev, td)).cpu().numpy().astype(np.float64)
    tol = 2e-6 if dtype == "float32" else 1e-13
    for b, p in enumerate(probs):
        op = oracle.SrmOperator(N, p.sign_bits, p.rows, p.perm)
        y_ref, x_ref = op.apply(X[b]), op.adjoint(W[b])
        assert np.linalg.norm(Yg[b] - y_ref) <= tol * np.linalg.norm(y_ref), b
        assert np.linalg.norm(Xg[b] - x_ref) <= tol * np.linalg.norm(x_ref), b


def test_perm_with_signs_matches_oracle(cs):
    """R diag(sigma) composed: sign bits and a permutation together (both tiers)."""
    dev = torch.device("cuda:0")
    for N, M in [(2048, 512), (65536, 16384)]:
        cfg = cs_inputs.Config(85, "sp", N, M, 8, "gauss", 0.0)
        probs = [cs_inputs.make_problem(cfg, b=b) for b in range(2)]
        for b, p in enumerate(probs):
            p.perm = cs_inputs.draw_perm(N, cs_inputs.rng(85, 0, b, 9))
        A = _op(cs, probs, dev, signs=True)
        X = np.random.default_rng(1).standard_normal((2, N))
        Yg = cs.cs_operator_apply(A, torch.from_numpy(X).to(dev, torch.float64)).cpu().numpy()
        for b, p in enumerate(probs):
            y_ref = oracle.SrmOperator(N, p.sign_bits, p.rows, p.perm).apply(X[b])
            assert np.linalg.norm(Yg[b] - y_ref) <= 1e-13 * np.linalg.norm(y_ref)


def test_non_permutation_rejected(cs):
    dev = torch.device("cuda:0")
    N, M = 256, 64
    _, probs = _probs(N, M, 4, 1)
    bits, rows = to_dev(probs, dev)
    bad = probs[0].perm.copy()
    bad[3] = bad[7]                       # a repeated value
    with pytest.raises(RuntimeError, match="permutation"):
        cs.Operator(N, M, None, rows, batch=1, perm=torch.from_numpy(bad[None]).to(dev))
    bad = probs[0].perm.copy()
    bad[0] = N                            # out of range
    with pytest.raises(RuntimeError, match="permutation"):
        cs.Operator(N, M, None, rows, batch=1, perm=torch.from_numpy(bad[None]).to(dev))


def _recover(cs, cfg, probs, dtype="float32", tol=None, ys=None):
    dev = torch.device("cuda:0")
    ys = measured(probs) if ys is None else ys
    A = _op(cs, probs, dev)
    td = getattr(torch, dtype)
    tol = tol if tol is not None else (1e-6 if dtype == "float32" else 1e-12)
    res = cs.cs_recover_batched(A, cfg.alg, torch.from_numpy(ys).to(dev, td), cfg.K, tol)
    torch.cuda.synchronize()
    return ys, res.support.cpu().numpy(), res.values.cpu().numpy().astype(np.float64), res.reports()


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_perm_recovery_small_ragged(cs, alg, dtype):
    cfg, probs = _probs(1024, 256, 16, 5, alg=alg, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, dtype)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-4 if dtype == "float32" else 1e-9)
    assert not bad, bad


def test_perm_recovery_c4_shape_batched(cs):
    """c4 shape (N = 16384, M = 4096, K = 256) with D F R: 32 problems, CTA tier."""
    cfg, probs = _probs(16384, 4096, 256, 32)
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad
    assert all(np.array_equal(np.sort(supp[b]), probs[b].support) for b in range(32))


def test_perm_recovery_grid_tier_fp64(cs):
    cfg, probs = _probs(65536, 16384, 1024, 1, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-8)
    assert not bad, bad


def test_perm_recovery_grid_tier_ompr_fp32(cs):
    cfg, probs = _probs(1 << 17, 1 << 15, 512, 1, alg="ompr")
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad


@pytest.mark.parametrize("alg,N,M,K", [("sp", 16384, 4096, 256), ("omp", 1024, 256, 8),
                                       ("cosamp", 2048, 512, 16), ("sp", 65536, 16384, 64)])
def test_perm_all_ties_go_to_lowest_original_index(cs, alg, N, M, K):
    """y = 0: every correlation ties at 0; the selected indices must be the lowest ORIGINAL
    indices (not the lowest transform positions), as in the oracle."""
    cfg, probs = _probs(N, M, K, 2, alg=alg)
    ys = np.zeros((2, M), dtype=np.float32)
    _, supp, vals, reps = _recover(cs, cfg, probs, ys=ys)
    refs = oracle_results(probs, ys)
    for b in range(2):
        assert np.array_equal(np.sort(supp[b]), refs[b].support), (alg, b)
