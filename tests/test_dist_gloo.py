"""Multi-rank path on CPU (gloo, world size 2): problem sharding and the result
gather bench.py runs over NCCL on GPUs.  The per-rank "recovery"
here is a stand-in that writes records derived from the global problem index, so
the test checks exactly the plumbing: which rank owns which problems, record
packing, and that rank 0 ends with every problem's record in problem order."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1509_03979_b200 import dist as csd  # noqa: E402

K = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_results(b0, count, dtype):
    idx = torch.arange(b0, b0 + count, dtype=torch.int64)
    supp = (idx[:, None] * 10 + torch.arange(K)[None, :]).to(torch.int32)
    vals = (idx[:, None].to(dtype) + torch.arange(K, dtype=dtype)[None, :] / 8)
    rep = (idx[:, None] % 251).to(torch.uint8).repeat(1, 40)
    return supp, vals, rep


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, cnt = csd.shard(total, rank, world)
        supp, vals, rep = _fake_results(b0, cnt, torch.float32)
        rec = csd.pack_records(supp, vals, rep)
        assert rec.shape == (cnt, csd.record_bytes(K, 4))
        allrec = csd.gather_records(rec, world, total=total)
        if rank == 0:
            s, v, r = csd.unpack_records(allrec, K, torch.float32)
            q.put((s.numpy(), v.numpy(), r.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_covers_every_problem_once():
    for total in [1, 7, 4096]:
        for world in [1, 2, 3, 8]:
            blocks = [csd.shard(total, r, world) for r in range(world)]
            covered = np.concatenate([np.arange(b0, b0 + c) for b0, c in blocks])
            assert np.array_equal(covered, np.arange(total))


def test_pack_unpack_roundtrip():
    supp, vals, rep = _fake_results(3, 4, torch.float64)
    s, v, r = csd.unpack_records(csd.pack_records(supp, vals, rep), K, torch.float64)
    assert torch.equal(s, supp) and torch.equal(v, vals) and torch.equal(r, rep)


@pytest.mark.parametrize("total", [64, 65])
def test_gloo_world2_gather_in_problem_order(total):
    """Equal blocks (the 4096 / G split of bench.py) and uneven ones (total % world != 0:
    the first rank holds one extra problem; gather_records pads and trims)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    s, v, r = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    es, ev, er = _fake_results(0, total, torch.float32)
    assert np.array_equal(s, es.numpy())
    assert np.array_equal(v, ev.numpy())
    assert np.array_equal(r, er.numpy())
