"""GPU parity of cs_recover / cs_recover_batched (OMP, SP, OMPR with the CG-solved
weighted LS) against the fp64 oracle on the same seeded inputs, through the C ABI.

Bar (BASELINE.json north_star): identical supports and
||s_gpu - s_oracle|| / ||s_oracle|| <= 1e-4 (fp32 GPU vs fp64 oracle)."""
import numpy as np
import pytest

import cs_inputs
import oracle
from cs_inputs import CONFIGS
from gpu_helpers import to_dev, perms_dev, measured, oracle_results, compare

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _run(cs, cfg, count, dtype="float32", tol=None, b0=0, opts=None):
    dev = torch.device("cuda:0")
    probs = cs_inputs.make_batch(cfg, b0=b0, count=count)
    ys = measured(probs)
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=count, perm=perms_dev(probs, dev))
    td = getattr(torch, dtype)
    if tol is None:
        tol = 1e-6 if dtype == "float32" else 1e-12
    Y = torch.from_numpy(ys).to(dev, td)
    res = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, tol, opts=opts)
    torch.cuda.synchronize()
    return probs, ys, res.support.cpu().numpy(), res.values.cpu().numpy(), res.reports()


def test_c1_omp_full_size(cs):
    cfg = CONFIGS[1]
    probs, ys, supp, vals, reps = _run(cs, cfg, 1)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad
    assert reps[0]["outer_iters"] == cfg.K
    assert reps[0]["termination"] == 0
    # noiseless: exact recovery of the planted signal as well
    assert np.array_equal(np.sort(supp[0]), probs[0].support)


def test_c4_sp_batched_full_size_sample(cs):
    cfg = CONFIGS[4]
    probs, ys, supp, vals, reps = _run(cs, cfg, 48)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad
    assert all(r["termination"] in (3, 4) for r in reps)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_small_ragged_batch_all_algs(cs, dtype):
    for alg in ["omp", "sp", "ompr", "cosamp"]:
        cfg = cs_inputs.Config(60, alg, 512, 128, 12, "gauss", 0.0)
        probs, ys, supp, vals, reps = _run(cs, cfg, 7, dtype)
        refs = oracle_results(probs, ys)
        bad, worst = compare(probs, refs, supp, vals, rtol=1e-4 if dtype == "float32" else 1e-9)
        assert not bad, (alg, bad)


def test_tiny_sizes(cs):
    for N, M, K, alg in [(8, 4, 1, "omp"), (16, 8, 2, "sp"), (32, 16, 3, "ompr"), (64, 32, 4, "sp"),
                         (16, 8, 2, "cosamp"), (64, 32, 4, "cosamp")]:
        cfg = cs_inputs.Config(61, alg, N, M, K, "pm1", 0.0)
        probs, ys, supp, vals, reps = _run(cs, cfg, 3, "float64")
        refs = oracle_results(probs, ys)
        bad, _ = compare(probs, refs, supp, vals, rtol=1e-9)
        assert not bad, (N, alg, bad)


def test_c2_sp_tier_l_scaled_fp64(cs):
    cfg = CONFIGS[2].scaled(2)          # N = 32768: Tier L (cooperative grid)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1, "float64", tol=1e-12)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-8)
    assert not bad, bad


def test_c3_ompr_tier_l_scaled(cs):
    cfg = CONFIGS[3].scaled(16)         # N = 65536, K = 512
    probs, ys, supp, vals, reps = _run(cs, cfg, 1)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad
    assert np.array_equal(np.sort(supp[0]), probs[0].support)


def test_c5_sp_tier_l_scaled_fp64(cs):
    cfg = CONFIGS[5].scaled(64)         # N = 2^18, K = 1024, compressible + noise
    probs, ys, supp, vals, reps = _run(cs, cfg, 1, "float64", tol=1e-12)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-8)
    assert not bad, bad


def test_deterministic_rerun(cs):
    cfg = CONFIGS[4].scaled(4, batch=8)
    a = _run(cs, cfg, 8)
    b = _run(cs, cfg, 8)
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[3], b[3])


@pytest.mark.parametrize("alg,N,M,K", [("omp", 1024, 256, 8), ("sp", 16384, 4096, 256),
                                       ("ompr", 2048, 512, 16), ("sp", 65536, 16384, 64),
                                       ("cosamp", 16384, 4096, 256), ("cosamp", 65536, 16384, 64)])
def test_all_ties_zero_measurements(cs, alg, N, M, K):
    """y = 0: every correlation is exactly 0, so every selection is a full tie and must
    go to the lowest indices; the oracle gives the same."""
    cfg = cs_inputs.Config(62, alg, N, M, K, "gauss", 0.0)
    probs = cs_inputs.make_batch(cfg, count=2)
    ys = np.zeros((2, M), dtype=np.float32)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(N, M, bits, rows, batch=2)
    res = cs.cs_recover_batched(A, alg, torch.from_numpy(ys).to(dev), K, 1e-6)
    torch.cuda.synchronize()
    supp = res.support.cpu().numpy()
    refs = oracle_results(probs, ys)
    for b in range(2):
        assert np.array_equal(np.sort(supp[b]), refs[b].support), (alg, b)
        assert np.array_equal(np.sort(supp[b]), np.arange(K))
    assert np.all(res.values.cpu().numpy() == 0)


def test_host_buffer_entry_point_matches_device_path(cs):
    """cs_recover_batched_host (chunked copy/compute pipeline) returns exactly what the
    device entry point returns, for a batch spanning several chunks and a ragged tail."""
    cfg = CONFIGS[4].scaled(4, batch=1300)     # N = 4096; chunks of 4 x #SM problems
    probs = cs_inputs.make_batch(cfg, count=1300)
    ys = measured(probs)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=1300)
    Yd = torch.from_numpy(ys).to(dev)
    ref = cs.cs_recover_batched(A, cfg.alg, Yd, cfg.K, 1e-6)
    host = cs.cs_recover_batched_host(A, cfg.alg, torch.from_numpy(ys).pin_memory(), cfg.K, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(host.support, ref.support.cpu())
    assert torch.equal(host.values, ref.values.cpu())
    assert np.array_equal(host.reports(), ref.reports())


@pytest.mark.parametrize("alg,N,M,K,dtype", [("sp", 16384, 4096, 1024, "float64"),
                                             ("omp", 8192, 2048, 512, "float64"),
                                             ("sp", 16384, 8192, 2048, "float32")])
def test_small_n_large_k_grid_fallback(cs, alg, N, M, K, dtype):
    """N <= 16384 whose pursuit does not fit one CTA's shared memory (fp64 with a large K,
    or a very large K) runs on the grid tier; it must still equal the oracle."""
    cfg = cs_inputs.Config(63, alg, N, M, K, "gauss", 0.0)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1, dtype)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-4 if dtype == "float32" else 1e-8)
    assert not bad, bad


@pytest.mark.parametrize("N,M,K", [(2048, 512, 16), (65536, 16384, 64)])
def test_nonfinite_measurements_flagged(cs, N, M, K):
    """y with a NaN / Inf: the report carries CS_DEV_NONFINITE_Y on both tiers,
    and the other problems of the batch are unaffected."""
    cfg = cs_inputs.Config(64, "sp", N, M, K, "gauss", 0.0)
    probs = cs_inputs.make_batch(cfg, count=2)
    ys = measured(probs)
    ys[1, 3] = np.nan
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(N, M, bits, rows, batch=2)
    res = cs.cs_recover_batched(A, "sp", torch.from_numpy(ys).to(dev), K, 1e-6)
    torch.cuda.synchronize()
    reps = res.reports()
    assert reps[1]["status"] & 1
    assert not (reps[0]["status"] & 1)
    refs = oracle_results(probs[:1], ys[:1])
    bad, _ = compare(probs[:1], refs, res.support.cpu().numpy()[:1], res.values.cpu().numpy()[:1])
    assert not bad, bad


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("cid,div", [(2, 2), (5, 64), (3, 16)])
def test_deterministic_rerun_grid_tier(cs, dtype, cid, div):
    """Fixed-order grid reductions and a deterministic order inside every support bucket
    (set_input_support ranks the atomically filled lists): repeated runs of the grid tier
    agree bit for bit — values, supports and every report field — in fp32 and fp64."""
    cfg = CONFIGS[cid].scaled(div)
    runs = [_run(cs, cfg, 1, dtype=dtype) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(runs[0][2], r[2])
        assert runs[0][3].tobytes() == r[3].tobytes()
        assert runs[0][4].tobytes() == r[4].tobytes()


# ---------------------------------------------------------------- CoSaMP (R33) ----
def test_cosamp_c4_shape_batched(cs):
    """CG-CoSaMP on the c4 workload shape (N = 16384, M = 4096, K = 256), CTA tier."""
    cfg = cs_inputs.Config(4, "cosamp", 16384, 4096, 256, "gauss", 0.0, batch=48)
    probs, ys, supp, vals, reps = _run(cs, cfg, 48)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad
    assert all(r["termination"] in (3, 4) for r in reps)
    assert all(np.array_equal(np.sort(supp[b]), probs[b].support) for b in range(48))


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_cosamp_noisy_ragged(cs, dtype):
    """Noisy K-sparse Gaussian signals, ragged batch of 5: fp64 equals the
    oracle; fp32 too at this size (well-separated coefficients)."""
    cfg = cs_inputs.Config(65, "cosamp", 2048, 768, 32, "gauss", 1e-3)
    probs, ys, supp, vals, reps = _run(cs, cfg, 5, dtype)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-4 if dtype == "float32" else 1e-9)
    assert not bad, bad


def test_cosamp_tier_l_fp64(cs):
    """Grid tier (N = 2^16): noisy c2-shape problem, fp64 against the oracle."""
    cfg = cs_inputs.Config(66, "cosamp", 65536, 16384, 1024, "gauss", 1e-2)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1, "float64", tol=1e-12)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-8)
    assert not bad, bad


def test_cosamp_tier_l_fp32_exact(cs):
    cfg = cs_inputs.Config(67, "cosamp", 1 << 18, 1 << 16, 2048, "gauss", 0.0)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad
    assert np.array_equal(np.sort(supp[0]), probs[0].support)


# ---------------------------------------------------------------- edge cases ------
@pytest.mark.parametrize("N", [1024, 65536])
@pytest.mark.parametrize("alg", ["omp", "sp"])
def test_full_sampling_m_equals_n(cs, N, alg):
    """M = N: every DCT row selected, A is orthogonal (A^T A = I) — one CG iteration
    solves each LS exactly; the recovery equals the oracle's on both tiers."""
    cfg = cs_inputs.Config(68, alg, N, N, 8, "gauss", 1e-2)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1, "float64")
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-9)
    assert not bad, bad


@pytest.mark.parametrize("alg", ["omp", "sp", "ompr", "cosamp"])
def test_k_equals_one(cs, alg):
    cfg = cs_inputs.Config(69, alg, 4096, 64, 1, "gauss", 0.0)
    probs, ys, supp, vals, reps = _run(cs, cfg, 3)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals)
    assert not bad, bad


def test_k_at_limit_n_over_2(cs):
    """K = N/2 (the ABI's upper bound) with OMPR (K + 1 <= M = N): a degenerate but legal call."""
    cfg = cs_inputs.Config(71, "ompr", 64, 64, 32, "gauss", 0.0)
    probs, ys, supp, vals, reps = _run(cs, cfg, 2, "float64")
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-8)
    assert not bad, bad


@pytest.mark.slow
def test_max_size_n_2_pow_25(cs):
    """N = 2^25 (the largest supported transform): noiseless SP recovers the planted support
    and is LS-optimal against the oracle operator (two fp64 applies; a whole oracle recovery
    at this size would take far too long)."""
    cfg = cs_inputs.Config(72, "sp", 1 << 25, 1 << 23, 1024, "gauss", 0.0)
    probs, ys, supp, vals, reps = _run(cs, cfg, 1)
    p = probs[0]
    assert np.array_equal(np.sort(supp[0]), p.support)
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows)
    s = np.zeros(p.N)
    s[supp[0]] = vals[0]
    assert np.linalg.norm(s - p.s) <= 1e-4 * np.linalg.norm(p.s)
    r = ys[0].astype(np.float64) - op.apply(s)
    assert np.linalg.norm(op.adjoint(r)[supp[0]]) <= 1e-4 * np.linalg.norm(op.adjoint(ys[0].astype(np.float64))[supp[0]])


@pytest.mark.parametrize("variant", ["perm", "psi", "dft"])
def test_host_buffer_entry_point_operator_variants(cs, variant):
    """The chunked host pipeline slices per-instance operator data (pi / pi^-1, the DFT
    position map; the shared all-rows instance of Psi) correctly: host results equal the
    device entry point's over several chunks and a ragged tail."""
    kw = {"perm": dict(randomizer="perm"), "psi": dict(randomizer="perm", psi="dct"),
          "dft": dict(randomizer="perm", transform="dft")}[variant]
    cfg = cs_inputs.Config(73, "sp", 2048, 512, 16, "gauss", 0.0, **kw)
    B = 1300
    probs = cs_inputs.make_batch(cfg, count=B)
    ys = measured(probs)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, probs[0].M, None, rows, batch=B, perm=perms_dev(probs, dev),
                    psi=("dct" if variant == "psi" else None), transform=probs[0].transform)
    Yd = torch.from_numpy(ys).to(dev)
    ref = cs.cs_recover_batched(A, cfg.alg, Yd, cfg.K, 1e-6)
    host = cs.cs_recover_batched_host(A, cfg.alg, torch.from_numpy(ys).pin_memory(), cfg.K, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(host.support, ref.support.cpu())
    assert torch.equal(host.values, ref.values.cpu())
    pick = [0, 517, 1299]
    sub = [probs[i] for i in pick]
    bad, _ = compare(sub, oracle_results(sub, ys[pick]), ref.support.cpu().numpy()[pick],
                     ref.values.cpu().numpy()[pick].astype(np.float64))
    assert not bad, bad


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batched_grid_tier_groups(cs, dtype):
    """A batch on the grid tier (N = 2^15) runs as several groups of blocks side by side, each
    with its own workspace slice and barrier: every instance equals the oracle."""
    cfg = cs_inputs.Config(75, "sp", 32768, 8192, 64, "gauss", 1e-3)
    probs, ys, supp, vals, reps = _run(cs, cfg, 7, dtype)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-4 if dtype == "float32" else 1e-8)
    assert not bad, bad
