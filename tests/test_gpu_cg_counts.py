"""Grid-tier CG (R37: one grid reduction per iteration, vector updates in the next H's
scatter) against Algorithm 1 as the oracle runs it: at fp64 and the same
tolerance on both sides, a whole recovery takes the same number of pursuit iterations and —
up to one CG iteration per solve where a residual sits at the threshold — the same number of
CG iterations.  A dropped update, a wrong alpha / beta or a stale direction changes these
counts by far more than the slack (the first R37 version, whose ||r||^2 ran as a recurrence,
diverged to 1e77 on c2)."""
import numpy as np
import pytest

import cs_inputs
import oracle
from gpu_helpers import to_dev, measured

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-12


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


CASES = [
    cs_inputs.Config(71, "sp", 1 << 15, 1 << 13, 1024, "gauss", 1e-3),
    cs_inputs.Config(72, "ompr", 1 << 15, 1 << 13, 256, "pm1", 0.0),
    cs_inputs.Config(73, "cosamp", 1 << 15, 1 << 13, 512, "gauss", 0.0),
    cs_inputs.Config(74, "omp", 1 << 15, 1 << 12, 48, "gauss", 0.0),
    cs_inputs.Config(75, "sp", 1 << 16, 1 << 14, 2048, "power", 1e-2),
]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: f"{c.alg}-N{c.N}-K{c.K}")
def test_grid_cg_iteration_counts_match_oracle(cs, cfg):
    dev = torch.device("cuda:0")
    probs = cs_inputs.make_batch(cfg, count=1)
    ys = measured(probs)
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=1)
    Y = torch.from_numpy(ys).to(dev, torch.float64)
    res = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, TOL)
    torch.cuda.synchronize()
    rep = res.reports()[0]
    p = probs[0]
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    ref = oracle.recover(p.alg, op, ys[0].astype(np.float64), p.K, tol=TOL)
    assert int(rep["outer_iters"]) == ref.outer_iters, (int(rep["outer_iters"]), ref.outer_iters)
    gpu_cg = int(rep["cg_iters_total"])
    assert abs(gpu_cg - ref.cg_iters) <= ref.outer_iters + 1, (gpu_cg, ref.cg_iters)
    np.testing.assert_array_equal(np.sort(res.support.cpu().numpy()[0]), ref.support)
