"""GPU parity of the single-signal distributed operator (NEXT-4, cs_dist_phase /
cs_dist_copy, paper_1509_03979_b200/dist.py): G logical ranks played by one process on one
GPU, host-sequenced (every phase of every rank completes before the exchange reads it; no
kernel waits on another), the all-to-all and the sums done by the emulated exchange.  The
distributed y = A x and x = A^T y must equal the oracle's (fp32 tolerance of
test_gpu_operator.py) and the single-GPU cs_operator_apply / _adjoint."""
import numpy as np
import pytest

import cs_inputs
import oracle
from gpu_helpers import to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _run(cs, N, M, world, seed=0):
    from paper_1509_03979_b200 import dist as csd
    dev = torch.device("cuda:0")
    cfg = cs_inputs.Config(90 + seed, "sp", N, M, max(1, M // 8), "gauss", 0.0)
    p = cs_inputs.make_problem(cfg, b=0)
    bits, rows = to_dev([p], dev)
    A = cs.Operator(N, M, bits, rows, batch=1)
    plan = csd.dist_plan(N, world)
    ranks = [csd.DistOperator(A, plan, r) for r in range(world)]
    g = np.random.default_rng(N + world)
    x = g.standard_normal(N)
    w = g.standard_normal(M)
    xd = torch.from_numpy(x).to(dev, torch.float32)
    wd = torch.from_numpy(w).to(dev, torch.float32)
    y = csd.dist_apply(ranks, xd, csd.emulated_exchange, csd.emulated_allreduce)
    xa = csd.dist_adjoint(ranks, wd, csd.emulated_exchange, csd.emulated_allreduce)
    y1 = cs.cs_operator_apply(A, xd[None])[0]
    x1 = cs.cs_operator_adjoint(A, wd[None])[0]
    torch.cuda.synchronize()
    return p, x, w, y.double().cpu().numpy(), xa.double().cpu().numpy(), y1.double().cpu().numpy(), \
        x1.double().cpu().numpy()


def _close_to_single(N, G, y, xa, y1, x1):
    """The ranks run the single-GPU passes on their tiles; the partial y / x they sum have
    disjoint supports, so the only differences are the exchange-free kernel's own fp32
    rounding (different code instances may contract differently): well inside 1e-6."""
    dy = np.linalg.norm(y - y1) / np.linalg.norm(y1)
    dx = np.linalg.norm(xa - x1) / np.linalg.norm(x1)
    print(f"N={N} G={G}: |y-y1|/|y1| {dy:.2e} exact {np.array_equal(y, y1)}, "
          f"|x-x1|/|x1| {dx:.2e} exact {np.array_equal(xa, x1)}")
    assert dy <= 1e-6 and dx <= 1e-6, (N, G, dy, dx)


def _worlds(cs, N):
    from paper_1509_03979_b200 import dist as csd
    p1 = csd.dist_plan(N, 1)
    nt = p1.L2 // p1.CT
    return [G for G in (1, 2, 3, 4, 8) if nt % G == 0]


@pytest.mark.parametrize("N", [1 << 15, 1 << 16, 1 << 18, 1 << 20])
def test_dist_matches_oracle(cs, N):
    M = N // 4
    for G in _worlds(cs, N):
        p, x, w, y, xa, y1, x1 = _run(cs, N, M, G)
        op = oracle.SrmOperator(N, p.sign_bits, p.rows)
        y_ref, x_ref = op.apply(x), op.adjoint(w)
        ey = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
        ex = np.linalg.norm(xa - x_ref) / np.linalg.norm(x_ref)
        assert ey <= 2e-6 and ex <= 2e-6, (N, G, ey, ex)
        _close_to_single(N, G, y, xa, y1, x1)


@pytest.mark.parametrize("N", [1 << 22, 1 << 24])
def test_dist_full_size_matches_single_gpu(cs, N):
    """c5's N = 2^24 (M = N / 4): distributed over G = 2, 4, 8 equals the single-GPU operator."""
    M = N // 4
    for G in [g for g in _worlds(cs, N) if g > 1]:
        _, _, _, y, xa, y1, x1 = _run(cs, N, M, G, seed=1)
        _close_to_single(N, G, y, xa, y1, x1)


def test_dist_rejects_small_and_bad_ranges(cs):
    from paper_1509_03979_b200 import dist as csd
    with pytest.raises(RuntimeError):
        csd.dist_plan(1 << 14, 2)      # Tier S size: no four-step intermediate
    with pytest.raises(ValueError):
        csd.dist_plan(1 << 15, 7)      # 7 does not divide the column tiles
