"""F = partial Fourier (the MRI case of D F R; SURVEY §8f NEXT-3,
DESIGN.md R36) on the CUDA path, through the C ABI (cs_operator_create_dft): operator and
adjoint against the fp64 oracle on both tiers, with and without the Eq.(7) permutation, the
device-side frequency check, and recovery parity for all four pursuits."""
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


def _probs(N, M, K, batch, alg="sp", randomizer="perm", noise=0.0, seed=0):
    cfg = cs_inputs.Config(87 + seed, alg, N, M, K, "gauss", noise, randomizer=randomizer, transform="dft")
    return cfg, [cs_inputs.make_problem(cfg, b=b) for b in range(batch)]


def _op(cs, probs, dev):
    bits, rows = to_dev(probs, dev)
    p = probs[0]
    return cs.Operator(p.N, p.M, bits if p.perm is None else None, rows, batch=len(probs),
                       perm=perms_dev(probs, dev), transform="dft")


@pytest.mark.parametrize("N,M,batch", [(8, 2, 2), (64, 24, 3), (1024, 256, 2), (16384, 4096, 2),
                                       (32768, 8192, 1), (1 << 18, 1 << 16, 1)])
@pytest.mark.parametrize("randomizer", ["sign", "perm"])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_dft_apply_adjoint_match_oracle(cs, N, M, batch, randomizer, dtype):
    dev = torch.device("cuda:0")
    _, probs = _probs(N, M, 1, batch, randomizer=randomizer)
    A = _op(cs, probs, dev)
    g = np.random.default_rng(N + 7)
    X, W = g.standard_normal((batch, N)), g.standard_normal((batch, probs[0].M))
    td = getattr(torch, dtype)
    Yg = cs.cs_operator_apply(A, torch.from_numpy(X).to(dev, td)).cpu().numpy().astype(np.float64)
    Xg = cs.cs_operator_adjoint(A, torch.from_numpy(W).to(dev, td)).cpu().numpy().astype(np.float64)
    tol = 2e-6 if dtype == "float32" else 1e-13
    for b, p in enumerate(probs):
        op = oracle.SrmOperator(N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
        y_ref, x_ref = op.apply(X[b]), op.adjoint(W[b])
        assert np.linalg.norm(Yg[b] - y_ref) <= tol * np.linalg.norm(y_ref), b
        assert np.linalg.norm(Xg[b] - x_ref) <= tol * np.linalg.norm(x_ref), b


def test_dft_bad_frequencies_rejected(cs):
    dev = torch.device("cuda:0")
    N = 256
    for bad in ([0, 5, 9], [3, 5, N // 2], [5, 5, 7]):
        rows = torch.tensor([bad], dtype=torch.int32, device=dev)
        with pytest.raises(RuntimeError):
            cs.Operator(N, 6, None, rows, batch=1, transform="dft")


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
def test_dft_recovery_small_ragged(cs, alg, dtype):
    cfg, probs = _probs(1024, 256, 16, 5, alg=alg, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, dtype)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-4 if dtype == "float32" else 1e-9)
    assert not bad, bad


def test_dft_recovery_c4_shape(cs):
    cfg, probs = _probs(16384, 4096, 256, 16)
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad
    assert all(np.array_equal(np.sort(supp[b]), probs[b].support) for b in range(16))


def test_dft_recovery_grid_tier_fp64(cs):
    cfg, probs = _probs(65536, 16384, 1024, 1, noise=1e-3)
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-8)
    assert not bad, bad


def test_dft_recovery_grid_tier_ompr_fp32(cs):
    cfg, probs = _probs(1 << 17, 1 << 15, 256, 1, alg="ompr")
    ys, supp, vals, reps = _recover(cs, cfg, probs)
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals)
    assert not bad, bad
    assert np.array_equal(np.sort(supp[0]), probs[0].support)


@pytest.mark.parametrize("N,M,K", [(2048, 512, 16), (65536, 16384, 64)])
def test_dft_all_ties_zero_measurements(cs, N, M, K):
    cfg, probs = _probs(N, M, K, 2)
    ys = np.zeros((2, M), dtype=np.float32)
    _, supp, vals, reps = _recover(cs, cfg, probs, ys=ys)
    refs = oracle_results(probs, ys)
    for b in range(2):
        assert np.array_equal(np.sort(supp[b]), refs[b].support)


@pytest.mark.parametrize("N,M,K,alg", [(16, 6, 1, "omp"), (32, 12, 2, "sp"), (64, 24, 3, "ompr"),
                                       (64, 30, 4, "cosamp"), (128, 48, 5, "sp")])
def test_dft_tiny_sizes_fp64(cs, N, M, K, alg):
    cfg, probs = _probs(N, M, K, 3, alg=alg)
    ys, supp, vals, reps = _recover(cs, cfg, probs, "float64")
    bad, _ = compare(probs, oracle_results(probs, ys), supp, vals, rtol=1e-9)
    assert not bad, bad
