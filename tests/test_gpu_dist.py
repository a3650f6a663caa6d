"""GPU parity of the single-signal distributed operator (NEXT-4, cs_dist_phase /
cs_dist_copy / cs_dist_row_offsets, paper_1509_03979_b200/dist.py): G logical ranks played
by one process on one GPU, host-sequenced (every phase of every rank is issued before the
exchange reads it, on one stream; no kernel waits on another), the all-to-all and the
all-gathers done by the emulated collectives.  The distributed y = A x and x = A^T y
(entered from and gathered to natural vectors through the layout phases) must equal the
oracle's (fp32 tolerance of test_gpu_operator.py) and the single-GPU cs_operator_apply /
_adjoint; A^T A x chained inside the distributed layouts must equal the single-GPU chain."""
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
    ex, ag = csd.emulated_exchange, csd.emulated_allgather
    yT = csd.dist_apply(ranks, [r.scatter_x(xd) for r in ranks], ex)
    y = csd.gather_y(ranks, yT, ag)[0]
    xa = csd.gather_x(ranks, csd.dist_adjoint(ranks, [r.scatter_y(wd) for r in ranks], ex), ag)[0]
    # A^T A x without leaving the distributed layouts (what an iterative solver chains)
    ata = csd.gather_x(ranks, csd.dist_adjoint(ranks, yT, ex), ag)[0]
    y1 = cs.cs_operator_apply(A, xd[None])[0]
    x1 = cs.cs_operator_adjoint(A, wd[None])[0]
    ata1 = cs.cs_operator_adjoint(A, y1[None])[0]
    torch.cuda.synchronize()
    h = lambda t: t.double().cpu().numpy()
    assert np.array_equal(h(ata), h(ata1)) or \
        np.linalg.norm(h(ata) - h(ata1)) <= 1e-6 * np.linalg.norm(h(ata1)), (N, world)
    return p, x, w, h(y), h(xa), h(y1), h(x1)


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


def _mp_worker(rank, world, port, N, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1509_03979_b200 as cs
        from paper_1509_03979_b200 import dist as csd
        dev = torch.device("cuda:0")
        M = N // 4
        cfg = cs_inputs.Config(95, "sp", N, M, M // 8, "gauss", 0.0)
        p = cs_inputs.make_problem(cfg, b=0)
        bits, rows = to_dev([p], dev)
        A = cs.Operator(N, M, bits, rows, batch=1)
        r = csd.DistOperator(A, csd.dist_plan(N, world), rank)
        ex, ag, _ = csd.process_group_exchange(host_staged=True)
        g = np.random.default_rng(7)
        xd = torch.from_numpy(g.standard_normal(N)).to(dev, torch.float32)
        yT = csd.dist_apply([r], [r.scatter_x(xd)], ex)
        y = csd.gather_y([r], yT, ag)[0]
        x2 = csd.gather_x([r], csd.dist_adjoint([r], yT, ex), ag)[0]
        y1 = cs.cs_operator_apply(A, xd[None])[0]
        x21 = cs.cs_operator_adjoint(A, y1[None])[0]
        torch.cuda.synchronize()
        q.put((rank, float((y - y1).norm() / y1.norm()), float((x2 - x21).norm() / x21.norm())))
    finally:
        dist.destroy_process_group()


def test_dist_two_processes_gloo_host_staged(cs):
    """Two real processes (torch.distributed, gloo, exchange staged through host memory; the
    ranks' kernels never wait on one another) running the distributed apply / adjoint."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, 2, port, 1 << 20, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank, ey, ex in res:
        assert ey <= 1e-6 and ex <= 1e-6, (rank, ey, ex)


def test_dist_phase_argument_errors(cs):
    """include/cs.h cs_dist_*: CS_ERR_INVALID_ARG for ranges out of bounds / missing buffers,
    CS_ERR_UNSUPPORTED for an operator the distributed path does not cover."""
    import ctypes
    from paper_1509_03979_b200 import dist as csd
    dev = torch.device("cuda:0")
    N, M = 1 << 16, 1 << 14
    cfg = cs_inputs.Config(97, "sp", N, M, 16, "gauss", 0.0)
    p = cs_inputs.make_problem(cfg, b=0)
    bits, rows = to_dev([p], dev)
    A = cs.Operator(N, M, bits, rows)
    lib = cs.load_library()
    plan = csd.dist_plan(N, 2)
    r = csd.DistOperator(A, plan, 0)
    P = ctypes.c_void_p
    ntiles = plan.L2 // plan.CT
    buf = torch.empty(N, device=dev)
    st = P(torch.cuda.current_stream().cuda_stream)
    ws, nb = P(r.ws.data_ptr()), r.ws.numel()
    INVALID, UNSUPPORTED = 1, 2
    bad = [
        (csd.DP_A, 0, ntiles + 1, 0, 1, buf, None),            # tile range past the end
        (csd.DP_A, 2, 1, 0, 1, buf, None),                     # t_hi < t_lo
        (csd.DP_BF, 0, 1, 0, plan.L1 // 2 + 2, None, buf),     # item range past the end
        (csd.DP_A, 0, 1, 0, 1, None, None),                    # missing input
        (csd.DP_C, 0, 1, 0, 1, None, None),                    # missing output
        (csd.DP_XG, 0, 3, 0, 1, buf, buf),                     # uneven split for the gather
        (csd.DP_XS, 0, 0, 0, 1, buf, buf),                     # empty column range
        (99, 0, 1, 0, 1, buf, buf),                            # unknown phase
    ]
    for ph, t0, t1, i0, i1, a, b in bad:
        rc = lib.cs_dist_phase(A.handle, ph, t0, t1, i0, i1, P(a.data_ptr()) if a is not None else None,
                               P(b.data_ptr()) if b is not None else None, ws, nb, st)
        assert rc == INVALID, (ph, t0, t1, i0, i1, rc)
    rc = lib.cs_dist_phase(A.handle, csd.DP_A, 0, 1, 0, 1, P(buf.data_ptr()), None, ws, 16, st)
    assert rc != 0                                            # workspace too small
    small = cs.Operator(4096, 1024, *to_dev([cs_inputs.make_problem(
        cs_inputs.Config(98, "sp", 4096, 1024, 8, "gauss", 0.0), b=0)], dev))
    rc = lib.cs_dist_phase(small.handle, csd.DP_A, 0, 1, 0, 1, P(buf.data_ptr()), None, ws, nb, st)
    assert rc == UNSUPPORTED
    off = (ctypes.c_int64 * (plan.L1 + 1))()
    assert lib.cs_dist_row_offsets(small.handle, off) == UNSUPPORTED
    assert lib.cs_dist_row_offsets(A.handle, off) == 0 and off[plan.L1] == M and list(off) == sorted(off)


def test_dist_graphs_match_eager(cs):
    """DistGraphs (each rank's halves captured as CUDA graphs, the exchange between them)
    gives the same y = A x and x = A^T y as the eager calls, bit for bit."""
    from paper_1509_03979_b200 import dist as csd
    dev = torch.device("cuda:0")
    N, M, G = 1 << 20, 1 << 18, 4
    cfg = cs_inputs.Config(96, "sp", N, M, 64, "gauss", 0.0)
    p = cs_inputs.make_problem(cfg, b=0)
    bits, rows = to_dev([p], dev)
    A = cs.Operator(N, M, bits, rows)
    plan = csd.dist_plan(N, G)
    ranks = [csd.DistOperator(A, plan, r) for r in range(G)]
    graphs = [csd.DistGraphs(r) for r in ranks]
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(N, generator=g).to(dev)
    w = torch.randn(M, generator=g).to(dev)
    ex, ag = csd.emulated_exchange, csd.emulated_allgather
    y_ref = csd.gather_y(ranks, csd.dist_apply(ranks, [r.scatter_x(x) for r in ranks], ex), ag)[0]
    xa_ref = csd.gather_x(ranks, csd.dist_adjoint(ranks, [r.scatter_y(w) for r in ranks], ex), ag)[0]
    for _ in range(2):                       # replays are repeatable
        for r, gr in zip(ranks, graphs):
            gr.x.copy_(r.scatter_x(x))
            gr.pre_apply.replay()
        recvs = ex([gr.send(0) for gr in graphs])
        for gr, buf in zip(graphs, recvs):
            gr.recv_buf(0).copy_(buf)
            gr.post_apply.replay()
        y = csd.gather_y(ranks, [gr.yT for gr in graphs], ag)[0]
        for r, gr in zip(ranks, graphs):
            gr.y_in.copy_(r.scatter_y(w))
            gr.pre_adjoint.replay()
        recvs = ex([gr.send(1) for gr in graphs])
        for gr, buf in zip(graphs, recvs):
            gr.recv_buf(1).copy_(buf)
            gr.post_adjoint.replay()
        xa = csd.gather_x(ranks, [gr.xc_out for gr in graphs], ag)[0]
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref) and torch.equal(xa, xa_ref)
