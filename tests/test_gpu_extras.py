"""The remaining boundary calls of SV §8(b): the dense output (cs_support_to_dense) and the
single-process multi-GPU results gather (cs_comm_init / cs_gather_batched / cs_comm_destroy).
One GPU here: the gather runs with one device (the root's own block, the same code path
that frames the NCCL send/recv of the other devices)."""
import numpy as np
import pytest

import cs_inputs
from gpu_helpers import to_dev, measured

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _recovery(cs, count=6):
    cfg = cs_inputs.Config(74, "sp", 1024, 256, 12, "gauss", 0.0)
    probs = cs_inputs.make_batch(cfg, count=count)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=count)
    res = cs.cs_recover_batched(A, "sp", torch.from_numpy(measured(probs)).to(dev), cfg.K, 1e-6)
    torch.cuda.synchronize()
    return cfg, probs, res


def test_support_to_dense(cs):
    cfg, probs, res = _recovery(cs)
    for dt in (torch.float32, torch.float64):
        dense = cs.cs_support_to_dense(res.support, res.values.to(dt), cfg.N).cpu().numpy()
        want = np.zeros((len(probs), cfg.N))
        s, v = res.support.cpu().numpy(), res.values.cpu().numpy()
        for b in range(len(probs)):
            want[b, s[b]] = v[b]
        np.testing.assert_array_equal(dense, want.astype(dense.dtype))
        # noiseless: the dense signal is the planted one (to fp32 resolution)
        for b, p in enumerate(probs):
            assert np.linalg.norm(dense[b] - p.s) <= 1e-5 * np.linalg.norm(p.s)


def test_comm_gather_single_device(cs):
    cfg, probs, res = _recovery(cs)
    comm = cs.Comm([0])
    supp, vals, reps = comm.gather([res], root=0)
    torch.cuda.synchronize()
    assert torch.equal(supp, res.support)
    assert torch.equal(vals, res.values)
    assert torch.equal(reps, res.report_dev)
    del comm


def test_comm_gather_ordered_after_producer_stream(cs):
    """cs_gather_batched_after (via Comm.gather, which passes torch's current streams): the
    recovery is enqueued and the gather issued with no host synchronisation in between; the
    gathered records are still the finished results (gather ordering)."""
    cfg = cs_inputs.CONFIGS[4].scaled(4, batch=64)
    probs = cs_inputs.make_batch(cfg, count=64)
    ys = measured(probs)
    dev = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=64)
    Y = torch.from_numpy(ys).to(dev)
    comm = cs.Comm([0])
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        res = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6, stream=side)
        supp, vals, reps = comm.gather([res], root=0)       # no synchronize before
    torch.cuda.synchronize()
    ref = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(supp, ref.support) and torch.equal(vals, ref.values)
    del comm


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_comm_gather_two_devices_matches_single_device(cs):
    """Two devices, NCCL send/recv into the root's arrays: the records equal a one-device run
    of the same problems (bit for bit)."""
    cfg = cs_inputs.CONFIGS[4].scaled(4, batch=32)
    probs = cs_inputs.make_batch(cfg, count=32)
    ys = measured(probs)
    out = []
    for d in (0, 1):
        dev = torch.device("cuda", d)
        with torch.cuda.device(d):
            bits, rows = to_dev(probs[16 * d:16 * d + 16], dev)
            A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=16)
            out.append(cs.cs_recover_batched(A, cfg.alg, torch.from_numpy(ys[16 * d:16 * d + 16]).to(dev),
                                             cfg.K, 1e-6))
    comm = cs.Comm([0, 1])
    supp, vals, reps = comm.gather(out, root=0)
    torch.cuda.synchronize()
    dev0 = torch.device("cuda:0")
    bits, rows = to_dev(probs, dev0)
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=32)
    ref = cs.cs_recover_batched(A, cfg.alg, torch.from_numpy(ys).to(dev0), cfg.K, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(supp, ref.support) and torch.equal(vals, ref.values)


def test_host_pipeline_more_than_64_chunks(cs):
    """A host-buffer batch larger than 64 chunks of two recovery waves (the chunk grows),
    equal to the device entry point bit for bit."""
    cfg = cs_inputs.Config(66, "sp", 256, 64, 4, "gauss", 0.0)
    B = 40000
    g = np.random.default_rng(66)
    bits = torch.from_numpy(cs_inputs.pack_sign_bits(g.integers(0, 2, (B, cfg.N)).astype(bool).reshape(-1))
                            .view(np.int32).reshape(B, -1)).cuda()
    rows = torch.from_numpy(np.stack([np.sort(g.choice(cfg.N, cfg.M, replace=False)) for _ in range(B)])
                            .astype(np.int32)).cuda()
    A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=B)
    Y = torch.from_numpy(g.standard_normal((B, cfg.M)).astype(np.float32))
    ref = cs.cs_recover_batched(A, cfg.alg, Y.cuda(), cfg.K, 1e-6)
    host = cs.cs_recover_batched_host(A, cfg.alg, Y.pin_memory(), cfg.K, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(host.support, ref.support.cpu())
    assert torch.equal(host.values, ref.values.cpu())
