"""Host logic of the single-signal distributed operator (NEXT-4, DESIGN.md §8.3,
paper_1509_03979_b200/dist.py) on CPU: the ownership plan partitions the four-step
intermediate, and the pack -> all-to-all -> unpack exchange leaves every rank holding exactly
what its next pass reads — row owners all columns of their rows after pass A, column owners
all rows of their columns after pass B.  The segment copy is a numpy stand-in for
cs_dist_copy's kernel (same segment definition, include/cs.h); the exchange is the
single-process emulation and, in the gloo test, torch.distributed's all_to_all_single."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1509_03979_b200 import dist as csd  # noqa: E402

GEOMS = [(8, 16, 4), (64, 128, 4), (16, 256, 8), (512, 1024, 4)]


def _truth(L1, L2):
    r = np.arange(L1)[:, None].astype(np.float32)
    c = np.arange(L2)[None, :].astype(np.float32)
    return np.stack([r * 4096 + c, -(r + 1) * (c + 1)], axis=-1)   # complex as (re, im) pairs


def _copy(wk, rows, col0, seg_len, buf=None):
    """cs_dist_copy stand-in: pack when buf is None (returns the flat buffer), else unpack."""
    if buf is None:
        return np.concatenate([wk[r, c:c + seg_len].reshape(-1) for r, c in zip(rows, col0)] or
                              [np.zeros(0, np.float32)])
    n = 2 * seg_len
    for k, (r, c) in enumerate(zip(rows, col0)):
        wk[r, c:c + seg_len] = buf[k * n:(k + 1) * n].reshape(seg_len, 2)


def _round(plan, wks, direction, exchange):
    sends = []
    for r in range(plan.world):
        rows, col0, counts = plan.segments(r, direction, True)
        _, _, rcounts = plan.segments(r, direction, False)
        buf = torch.from_numpy(_copy(wks[r], rows, col0, plan.seg_len))
        sends.append((buf, [2 * c * plan.seg_len for c in counts], [2 * c * plan.seg_len for c in rcounts]))
    recvs = exchange(sends)
    for r in range(plan.world):
        rows, col0, _ = plan.segments(r, direction, False)
        _copy(wks[r], rows, col0, plan.seg_len, recvs[r].numpy())


@pytest.mark.parametrize("L1,L2,CT", GEOMS)
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_partitions_rows_columns_items(L1, L2, CT, world):
    if (L2 // CT) % world:
        with pytest.raises(ValueError):
            csd.DistPlan(2 * L1 * L2, world, L1, L2, CT)
        return
    p = csd.DistPlan(2 * L1 * L2, world, L1, L2, CT)
    assert sorted(sum(p.rows, [])) == list(range(L1))            # every row once
    cols = np.concatenate([np.arange(a, b) for a, b in p.cols])
    assert np.array_equal(cols, np.arange(L2))                  # every column once, in order
    assert p.items[0][0] == 0 and p.items[-1][1] == L1 // 2 + 1
    for r in range(world):
        for i in range(*p.items[r]):                              # the DCT split's pair (i, L1 - i)
            assert i in p.rows[r] and (L1 - i) % L1 in p.rows[r]
        assert p.cols[r][1] - p.cols[r][0] == p.seg_len


@pytest.mark.parametrize("L1,L2,CT", GEOMS)
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_exchange_delivers_rows_then_columns(L1, L2, CT, world):
    if (L2 // CT) % world:
        pytest.skip("world does not divide the column tiles")
    p = csd.DistPlan(2 * L1 * L2, world, L1, L2, CT)
    T = _truth(L1, L2)
    # after pass A: rank r holds only its columns
    wks = []
    for r in range(world):
        w = np.full_like(T, np.nan)
        a, b = p.cols[r]
        w[:, a:b] = T[:, a:b]
        wks.append(w)
    _round(p, wks, 0, csd.emulated_exchange)
    for r in range(world):
        assert np.array_equal(wks[r][p.rows[r]], T[p.rows[r]])
    # after pass B: rank r holds only its rows (new values); the exchange returns its columns
    T2 = T * 3 + 1
    wks = []
    for r in range(world):
        w = np.full_like(T, np.nan)
        w[p.rows[r]] = T2[p.rows[r]]
        wks.append(w)
    _round(p, wks, 1, csd.emulated_exchange)
    for r in range(world):
        a, b = p.cols[r]
        assert np.array_equal(wks[r][:, a:b], T2[:, a:b])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L1, L2, CT = 64, 128, 4
        p = csd.DistPlan(2 * L1 * L2, world, L1, L2, CT)
        exchange, allgather, allreduce = csd.process_group_exchange()
        T = _truth(L1, L2)
        ok = True
        for direction in (0, 1):
            w = np.full_like(T, np.nan)
            if direction == 0:
                a, b = p.cols[rank]
                w[:, a:b] = T[:, a:b]
            else:
                w[p.rows[rank]] = T[p.rows[rank]]
            rows, col0, counts = p.segments(rank, direction, True)
            _, _, rcounts = p.segments(rank, direction, False)
            buf = torch.from_numpy(_copy(w, rows, col0, p.seg_len))
            (recv,) = exchange([(buf, [2 * c * p.seg_len for c in counts], [2 * c * p.seg_len for c in rcounts])])
            rows, col0, _ = p.segments(rank, direction, False)
            _copy(w, rows, col0, p.seg_len, recv.numpy())
            if direction == 0:
                ok &= np.array_equal(w[p.rows[rank]], T[p.rows[rank]])
            else:
                a, b = p.cols[rank]
                ok &= np.array_equal(w[:, a:b], T[:, a:b])
        # the collectives of the layout changes (gather_x / gather_y)
        t = torch.full((5,), float(rank + 1))
        ok &= bool(torch.equal(allreduce([t]), torch.full((5,), float(world * (world + 1) // 2))))
        (g,) = allgather([torch.full((3,), float(rank))])
        ok &= bool(torch.equal(g, torch.tensor([0.0, 0, 0, 1, 1, 1])))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("L1,L2,CT", GEOMS)
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_y_ranges_partition_the_measurements(L1, L2, CT, world):
    """Rows of the transposed order hold consecutive yT entries (row_offsets); the ranks' row
    blocks cover every row once, so their yT ranges partition [0, M)."""
    if (L2 // CT) % world:
        pytest.skip("world does not divide the column tiles")
    p = csd.DistPlan(2 * L1 * L2, world, L1, L2, CT)
    rng = np.random.default_rng(L1 + world)
    counts = rng.integers(0, 2 * L2 + 1, size=L1)            # selected entries per row
    offs = np.concatenate([[0], np.cumsum(counts)]).tolist()
    covered = np.zeros(offs[-1], np.int64)
    for r in range(world):
        rows = set()
        for a, b in p.y_ranges(r, offs):
            covered[a:b] += 1
            rows |= {k for k in range(L1) if offs[k] >= a and offs[k + 1] <= b and counts[k] > 0}
        assert rows == {k for k in p.rows[r] if counts[k] > 0}
    assert np.all(covered == 1)
