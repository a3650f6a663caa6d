"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

Where the oracle finishes a whole recovery in seconds (c1, c2, c4 per problem) the
GPU result is compared with it outright; where it does not (c3: ~10-15 min, c5:
~7 min of fp64 CPU work) the full-size run is checked on properties that pin the
answer at any size:
  * noiseless exact recovery — the support is the planted one;
  * LS optimality on the returned support (Theorems 1-2): the residual
    is orthogonal to the selected columns, ||A_S^T (y - A_S x)|| <= eps ||A_S^T y||,
    evaluated with the ORACLE operator in fp64;
  * coefficients equal the oracle's CG-solved LS on that support (c3).
c3 and c5 are ALSO held to the oracle's own full-size answer: tools/oracle_reference.py
(oracle/ only) ran the fp64 oracle once on the same seeded inputs and stored support,
coefficients and iteration counts in tests/golden/oracle_c{3,5}.npz; the fp32 / fp64 GPU
results are compared with those (the y fed to the GPU is checked to be the y the oracle saw).
"""
import hashlib
import os

import numpy as np
import pytest

import cs_inputs
import oracle
from cs_inputs import CONFIGS
from gpu_helpers import to_dev, measured, oracle_results, compare, compare_fp32_floor, dense_from

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _recover(cs, cfg, probs, ys, dtype, tol):
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=len(probs))
    Y = torch.from_numpy(ys).to(dev, getattr(torch, dtype))
    res = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, tol)
    torch.cuda.synchronize()
    return res.support.cpu().numpy(), res.values.cpu().numpy().astype(np.float64), res.reports()


def _ls_optimality(p, y, supp, vals):
    """||A_S^T (y - A x)|| / ||A_S^T y|| with the oracle operator (fp64)."""
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    x = dense_from(p.N, supp, vals)
    r = y.astype(np.float64) - op.apply(x)
    g = op.adjoint(r)[supp]
    b = op.adjoint(y.astype(np.float64))[supp]
    return float(np.linalg.norm(g) / np.linalg.norm(b))


def test_c4_full_batch_sampled(cs):
    """The bench workload (4096 problems, one launch); 16 sampled problems vs the oracle."""
    cfg = CONFIGS[4]
    probs = cs_inputs.make_batch(cfg)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float32", 1e-6)
    rng = np.random.default_rng(4)
    pick = np.sort(rng.choice(cfg.batch, 16, replace=False))
    sub = [probs[i] for i in pick]
    refs = oracle_results(sub, ys[pick])
    bad, worst = compare(sub, refs, supp[pick], vals[pick])
    assert not bad, bad
    # every problem: a full, ascending support and a finished pursuit
    assert np.all(np.diff(supp, axis=1) > 0)
    assert np.all(np.isin(reps["termination"], (3, 4)))
    # noiseless: exact recovery for almost every problem.  A problem whose
    # planted support holds a coefficient below fp32 resolution (|s_j| ~ 1e-5 of
    # ||s||; ~1e-5 of Gaussian draws) can stop one SP iteration early in fp32 with
    # that index swapped (the fp64 path matches the oracle on all 4096): accepted
    # only under compare_fp32_floor's rule.
    planted = np.stack([p.support for p in probs])
    miss = np.nonzero(~(supp == planted).all(axis=1))[0]
    print(f"c4 fp32: {miss.size} of {cfg.batch} problems off the planted support: {miss.tolist()}")
    assert miss.size <= cfg.batch // 100, miss.size
    if miss.size:
        sub = [probs[i] for i in miss]
        refs = oracle_results(sub, ys[miss])
        bad = compare_fp32_floor(sub, refs, supp[miss], vals[miss])
        assert not bad, bad


def test_c4_full_batch_fp64_matches_oracle_everywhere_sampled(cs):
    """fp64 path on the whole 4096 batch: planted support on every problem (the oracle
    recovers it on every problem checked), 16 sampled problems equal to the oracle."""
    cfg = CONFIGS[4]
    probs = cs_inputs.make_batch(cfg)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float64", 1e-12)
    planted = np.stack([p.support for p in probs])
    assert (supp == planted).all()
    pick = np.sort(np.random.default_rng(5).choice(cfg.batch, 16, replace=False))
    sub = [probs[i] for i in pick]
    bad, worst = compare(sub, oracle_results(sub, ys[pick]), supp[pick], vals[pick], rtol=1e-9)
    assert not bad, bad


def test_c2_full_fp64_matches_oracle(cs):
    cfg = CONFIGS[2]
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float64", 1e-12)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-8)
    assert not bad, bad


def test_c2_full_fp32_matches_oracle(cs):
    """fp32 on the noisy c2 (SURVEY App. A flags ~15% of seeds as precision-fragile at a
    boundary index): on the BASELINE seed the fp32 GPU run ends on exactly the oracle's
    support, with coefficients within the BASELINE bar, and is LS-optimal at its CG floor."""
    cfg = CONFIGS[2]
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float32", 1e-6)
    refs = oracle_results(probs, ys)
    bad, worst = compare(probs, refs, supp, vals, rtol=1e-4)
    print(f"c2 fp32 vs oracle: symdiff {np.setxor1d(supp[0], refs[0].support).size}, rel {worst:.3e}")
    assert not bad, bad
    assert _ls_optimality(probs[0], ys[0], supp[0], vals[0]) < 5e-5


def test_c3_full_exact_recovery(cs):
    """OMPR(1) at N = 2^20: planted support recovered; coefficients equal the oracle's
    CG-solved LS on that support (rel <= 1e-4)."""
    cfg = CONFIGS[3]
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float32", 1e-6)
    p = probs[0]
    assert np.array_equal(supp[0], p.support)
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    c0 = op.adjoint(ys[0].astype(np.float64))
    ls = oracle.cg(op, p.support, c0, tol=1e-10)
    s_or = dense_from(p.N, p.support, ls.x)
    s_gpu = dense_from(p.N, supp[0], vals[0])
    assert np.linalg.norm(s_gpu - s_or) / np.linalg.norm(s_or) <= 1e-4
    assert reps[0]["termination"] == 3  # support fixed point


@pytest.mark.slow
def test_c5_full_fp64_ls_optimal(cs):
    """SP at N = 2^24, K = 65536, compressible + noise, fp64: LS-optimal on its support
    (to the fp64 CG tolerance) and a finished pursuit; the fp32 run overlaps it."""
    cfg = CONFIGS[5]
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float64", 1e-12)
    assert np.all(np.diff(supp[0]) > 0)
    assert reps[0]["termination"] in (3, 4)
    assert _ls_optimality(probs[0], ys[0], supp[0], vals[0]) < 1e-9
    s32, v32, r32 = _recover(cs, cfg, probs, ys, "float32", 1e-6)
    overlap = np.intersect1d(s32[0], supp[0]).size / cfg.K
    assert overlap >= 0.9, overlap   # fp32 diverges on the noise-dominated tail
    assert _ls_optimality(probs[0], ys[0], s32[0], v32[0]) < 1e-4


# ---- c3 / c5 against the oracle's full-size answer (tests/golden, tools/oracle_reference.py)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(cid):
    g = np.load(os.path.join(GOLDEN, f"oracle_c{cid}.npz"))
    return {k: g[k] for k in g.files}


def _same_input(cfg, ys, g):
    y_sha = hashlib.sha256(np.ascontiguousarray(ys[0], dtype=np.float32).tobytes()).hexdigest()
    assert y_sha == str(g["y_sha"]), "the GPU must see the y the oracle reference was computed on"


def _vs_golden(cfg, supp, vals, g):
    sg = np.sort(supp[0])
    symdiff = int(np.setxor1d(sg, g["support"]).size)
    s_or = dense_from(cfg.N, g["support"], g["x"])
    s_gpu = dense_from(cfg.N, supp[0], vals[0])
    rel = float(np.linalg.norm(s_gpu - s_or) / np.linalg.norm(s_or))
    return symdiff, rel


@pytest.mark.parametrize("dtype,tol,rtol", [("float32", 1e-6, 1e-4), ("float64", 1e-10, 1e-8)])
def test_c3_full_matches_oracle_reference(cs, dtype, tol, rtol):
    """OMPR(1) at N = 2^20 (the paper's P:89 size): the oracle's 698-swap trajectory ends on
    the planted support; the GPU (fp32 at the BASELINE bar, fp64 at the oracle's tol to
    1e-8) returns the same support and coefficients after the same number of swaps."""
    cfg = CONFIGS[3]
    g = _golden(3)
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    _same_input(cfg, ys, g)
    supp, vals, reps = _recover(cs, cfg, probs, ys, dtype, tol)
    symdiff, rel = _vs_golden(cfg, supp, vals, g)
    print(f"c3 {dtype} vs oracle: symdiff {symdiff}, rel {rel:.3e}, outer {reps[0]['outer_iters']} "
          f"(oracle {int(g['outer_iters'])}), cg {reps[0]['cg_iters_total']} (oracle {int(g['cg_iters'])})")
    assert symdiff == 0 and rel <= rtol, (symdiff, rel)
    assert reps[0]["outer_iters"] == int(g["outer_iters"])
    assert reps[0]["termination"] == int(g["termination"])


@pytest.mark.slow
def test_c5_full_fp64_matches_oracle_reference(cs):
    """SP at N = 2^24, K = 65536, compressible + noise (Table IV's largest N): the
    fp64 GPU path at the oracle's tolerance ends on the oracle's support (all 65536 indices,
    most of them noise-dominated) with coefficients within 1e-8, the same outer iterations
    and the same halting reason."""
    cfg = CONFIGS[5]
    g = _golden(5)
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    _same_input(cfg, ys, g)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float64", 1e-10)
    symdiff, rel = _vs_golden(cfg, supp, vals, g)
    print(f"c5 fp64 vs oracle: symdiff {symdiff}, rel {rel:.3e}, outer {reps[0]['outer_iters']} "
          f"(oracle {int(g['outer_iters'])}), term {reps[0]['termination']} (oracle {int(g['termination'])})")
    assert symdiff == 0 and rel <= 1e-8, (symdiff, rel)
    assert reps[0]["outer_iters"] == int(g["outer_iters"])
    assert reps[0]["termination"] == int(g["termination"])


@pytest.mark.slow
def test_c5_full_fp32_reported_against_oracle_reference(cs):
    """fp32 at c5 cannot match the oracle index for index (the tail of the
    power-law signal sits under the noise, below the fp32 LS floor).  Measured and printed:
    the support symmetric difference and coefficient rel-diff against the oracle's answer;
    held to: a finished pursuit, LS optimality on its own support, and the large coefficients
    (every index with |s_or| above the noise floor sigma sqrt(N/M)) all selected."""
    cfg = CONFIGS[5]
    g = _golden(5)
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    supp, vals, reps = _recover(cs, cfg, probs, ys, "float32", 1e-6)
    symdiff, rel = _vs_golden(cfg, supp, vals, g)
    print(f"c5 fp32 vs oracle: symdiff {symdiff} of {2 * cfg.K}, rel {rel:.3e}, "
          f"outer {reps[0]['outer_iters']} (oracle {int(g['outer_iters'])})")
    assert reps[0]["termination"] in (3, 4)
    assert _ls_optimality(probs[0], ys[0], supp[0], vals[0]) < 1e-4
    floor = cfg.noise * np.sqrt(cfg.N / cfg.M)
    big = g["support"][np.abs(g["x"]) > 10 * floor]
    assert np.isin(big, supp[0]).all()
    assert rel < 0.1     # measured 5.0e-2 (symdiff 8892 of 131072)


def test_c4_full_batch_fp32_refined_matches_oracle_everywhere(cs):
    """Mixed precision policy (cs_options.refine_fp64): the fp32 batch, with every
    problem whose fp32 result holds a coefficient below the fp32 resolution floor recovered
    again in fp64.  Every one of the 4096 problems then ends on the planted support (the fp64
    oracle's answer on each of them); the refined ones carry
    CS_DEV_REFINED_FP64 and equal the oracle to the fp64 bar; 16 sampled others equal the
    oracle to the fp32 bar."""
    cfg = CONFIGS[4]
    probs = cs_inputs.make_batch(cfg)
    ys = measured(probs)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=len(probs))
    opts = cs.cs_options()
    opts.refine_fp64 = 1
    res = cs.cs_recover_batched(A, cfg.alg, torch.from_numpy(ys).to(dev), cfg.K, 1e-6, opts=opts)
    torch.cuda.synchronize()
    supp, vals, reps = res.support.cpu().numpy(), res.values.cpu().numpy().astype(np.float64), res.reports()
    refined = np.nonzero(reps["status"] & 8)[0]
    print(f"c4 fp32 + fp64 refine: {refined.size} problems refined; "
          f"not refined (cap) {int(np.count_nonzero(reps['status'] & 16))}")
    planted = np.stack([p.support for p in probs])
    assert (supp == planted).all()
    assert 0 < refined.size <= 256
    sub = [probs[i] for i in refined[:12]]
    bad, worst = compare(sub, oracle_results(sub, ys[refined[:12]]), supp[refined[:12]], vals[refined[:12]], rtol=1e-6)
    assert not bad, bad
    pick = np.sort(np.random.default_rng(6).choice(cfg.batch, 16, replace=False))
    sub = [probs[i] for i in pick]
    bad, worst = compare(sub, oracle_results(sub, ys[pick]), supp[pick], vals[pick])
    assert not bad, bad


def test_c4_full_batch_host_pipeline_refined_equals_device_path(cs):
    """cs_options.refine_fp64 through the host-buffer entry point (fp32 chunks, then one
    refinement over the whole batch, results copied out after it) returns exactly what the
    device-path call returns: the same refined problems, bit-identical supports, values and
    reports."""
    cfg = CONFIGS[4]
    probs = cs_inputs.make_batch(cfg)
    ys = measured(probs)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=len(probs))
    opts = cs.cs_options()
    opts.refine_fp64 = 1
    ref = cs.cs_recover_batched(A, cfg.alg, torch.from_numpy(ys).to(dev), cfg.K, 1e-6, opts=opts)
    host = cs.cs_recover_batched_host(A, cfg.alg, torch.from_numpy(ys).pin_memory(), cfg.K, 1e-6, opts=opts)
    torch.cuda.synchronize()
    reps_h, reps_d = host.reports(), ref.reports()
    assert np.count_nonzero(reps_h["status"] & 8) == np.count_nonzero(reps_d["status"] & 8) > 0
    assert torch.equal(host.support, ref.support.cpu())
    assert torch.equal(host.values, ref.values.cpu())
    assert np.array_equal(reps_h, reps_d)
