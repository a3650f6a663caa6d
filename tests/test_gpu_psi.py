"""Dictionary Psi = DCT (A = Phi Psi, x = Psi s; "Psi is chosen to be a discrete
cosine transform", R35) on the CUDA path, through the
C ABI (cs_operator_create_ex): operator and adjoint against the fp64 oracle, with and
without the Eq.(7) permutation, on both tiers, and recovery parity for all four pursuits
(CTA tier; grid tier for N > 2^14 and for pursuits that do not fit one CTA)."""
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


def _probs(N, M, K, batch, alg="sp", randomizer="sign", noise=0.0, seed=0):
    cfg = cs_inputs.Config(86 + seed, alg, N, M, K, "gauss", noise, randomizer=randomizer, psi="dct")
    return cfg, [cs_inputs.make_problem(cfg, b=b) for b in range(batch)]


def _op(cs, probs, dev):
    bits, rows = to_dev(probs, dev)
    return cs.Operator(probs[0].N, probs[0].M, bits, rows, batch=len(probs),
                       perm=perms_dev(probs, dev), psi="dct")


@pytest.mark.parametrize("N,M,batch", [(8, 4, 2), (64, 16, 3), (1024, 256, 2), (16384, 4096, 2),
                                       (32768, 8192, 1), (1 << 18, 1 << 16, 1)])
@pytest.mark.parametrize("randomizer", ["sign", "perm"])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_psi_apply_adjoint_match_oracle(cs, N, M, batch, randomizer, dtype):
    dev = torch.device("cuda:0")
    _, probs = _probs(N, M, max(1, M // 8), batch, randomizer=randomizer)
    A = _op(cs, probs, dev)
    g = np.random.default_rng(N + 5)
    X, W = g.standard_normal((batch, N)), g.standard_normal((batch, M))
    td = getattr(torch, dtype)
    Yg = cs.cs_operator_apply(A, torch.from_numpy(X).to(dev, td)).cpu().numpy().astype(np.float64)
    Xg = cs.cs_operator_adjoint(A, torch.from_numpy(W).to(dev, td)).cpu().numpy().astype(np.float64)
    tol = 4e-6 if dtype == "float32" else 1e-13
    for b, p in enumerate(probs):
        op = oracle.SrmOperator(N, p.sign_bits, p.rows, p.perm, p.psi)
        y_ref, x_ref = op.apply(X[b]), op.adjoint(W[b])
        assert np.linalg.norm(Yg[b] - y_ref) <= tol * np.linalg.norm(y_ref), b
        assert np.linalg.norm(Xg[b] - x_ref) <= tol * np.linalg.norm(x_ref), b


def _recover(cs, cfg, probs, dtype="float32", ys=None, tol=None):
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
def test_psi_recovery_small_ragged(cs, alg, dtype):
    cfg, probs = _probs(1024, 256, 16, 5, alg=alg, randomizer="perm", noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, dtype)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-4 if dtype == "float32" else 1e-9)
    assert not bad, bad


def test_psi_recovery_c4_shape(cs):
    """c4 shape (N = 16384, M = 4096, K = 256) with A = Phi C_N: 16 problems vs the oracle,
    planted DCT-domain support recovered."""
    cfg, probs = _probs(16384, 4096, 256, 16)
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad
    assert all(np.array_equal(np.sort(supp[b]), probs[b].support) for b in range(16))


@pytest.mark.parametrize("alg", ["sp", "omp"])
def test_psi_all_ties_zero_measurements(cs, alg):
    cfg, probs = _probs(2048, 512, 16, 2, alg=alg, randomizer="perm")
    ys = np.zeros((2, 512), dtype=np.float32)
    _, supp, vals, reps = _recover(cs, cfg, probs, ys=ys)
    refs = oracle_results(probs, ys)
    for b in range(2):
        assert np.array_equal(np.sort(supp[b]), refs[b].support)


def test_psi_recovery_small_n_on_grid_tier_fp64(cs):
    """fp64 with a large K does not fit one CTA's shared memory: the grid tier runs it."""
    cfg, probs = _probs(16384, 8192, 2048, 1, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-8)
    assert not bad, bad


@pytest.mark.parametrize("randomizer", ["sign", "perm"])
def test_psi_recovery_grid_tier_fp64(cs, randomizer):
    cfg, probs = _probs(65536, 16384, 1024, 1, randomizer=randomizer, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-8)
    assert not bad, bad


def test_psi_recovery_grid_tier_ompr_fp32(cs):
    cfg, probs = _probs(1 << 17, 1 << 15, 256, 1, alg="ompr", randomizer="perm")
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad
    assert np.array_equal(np.sort(supp[0]), probs[0].support)


@pytest.mark.parametrize("N,M,K,alg", [(16, 8, 2, "sp"), (32, 16, 3, "ompr"), (64, 32, 4, "omp"),
                                       (64, 32, 4, "cosamp")])
def test_psi_tiny_sizes_fp64(cs, N, M, K, alg):
    cfg, probs = _probs(N, M, K, 3, alg=alg, randomizer="perm")
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-9)
    assert not bad, bad
