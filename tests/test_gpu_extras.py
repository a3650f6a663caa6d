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
