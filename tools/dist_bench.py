"""Per-rank cost of the distributed single-signal operator (NEXT-4) on one
B200: G logical ranks are host-sequenced on one GPU, so each rank's kernels run alone and
their CUDA-event time is that rank's compute on its own GPU.  Prints, per N and G: the
single-GPU apply / adjoint (cs_operator_apply / _adjoint), the slowest rank's compute per
application (phase + pack + unpack + phase), the bytes each rank sends in the all-to-all,
and the all-to-all time that NVLink 5 (900 GB/s per direction) would add at that size."""
import json
import sys
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402
g.build()
import paper_1509_03979_b200 as cs  # noqa: E402
from paper_1509_03979_b200 import dist as csd  # noqa: E402
import cs_inputs  # noqa: E402

dev = torch.device("cuda:0")
REPS = 20


def ev():
    return torch.cuda.Event(enable_timing=True)


def med(xs):
    return float(np.median(xs))


rows_out = []
for e in [int(a) for a in (sys.argv[1:] or ["22", "24", "25", "26"])]:
    N = 1 << e
    M = N // 4
    cfg = cs_inputs.Config(99, "sp", N, M, 16, "gauss", 0.0)
    rng = np.random.default_rng(e)
    sign = rng.integers(0, 2**32, size=(1, (N + 31) // 32), dtype=np.uint64).astype(np.uint32)
    rows = np.sort(rng.choice(N, size=M, replace=False)).astype(np.int32)[None]
    A = cs.Operator(N, M, torch.from_numpy(sign.view(np.int32)).to(dev), torch.from_numpy(rows).to(dev))
    x = torch.randn(1, N, device=dev)
    w = torch.randn(1, M, device=dev)
    # single GPU
    t1a, t1t = [], []
    for _ in range(REPS):
        a, b, c = ev(), ev(), ev()
        a.record(); cs.cs_operator_apply(A, x); b.record(); cs.cs_operator_adjoint(A, w); c.record()
        torch.cuda.synchronize()
        t1a.append(a.elapsed_time(b) * 1e3); t1t.append(b.elapsed_time(c) * 1e3)
    for G in [1, 2, 4, 8]:
        plan = csd.dist_plan(N, G)
        ranks = [csd.DistOperator(A, plan, r) for r in range(G)]
        xcs = [r.scatter_x(x[0]) for r in ranks]
        yTs = [r.scatter_y(w[0]) for r in ranks]
        ta = np.zeros((REPS, G)); tt = np.zeros((REPS, G)); pa = np.zeros((REPS, 4))
        sent = max(sum(r.seg[(0, True)][2]) - r.seg[(0, True)][2][i] for i, r in enumerate(ranks)) * 4
        for it in range(REPS):
            # apply: rank phases with their pack / unpack, timed per rank
            evs = []
            sends = []
            for r, xc in zip(ranks, xcs):
                a = ev(); a.record()
                r.phase(csd.DP_A, inp=xc)
                m = ev(); m.record()
                s = r.send_buffer(0)
                b = ev(); b.record()
                evs.append([a, b, m]); sends.append(s)
            recvs = csd.emulated_exchange(sends)
            yT = []
            for k, (r, buf) in enumerate(zip(ranks, recvs)):
                a = ev(); a.record()
                r.copy(0, False, buf)
                m = ev(); m.record()
                yT.append(r.phase(csd.DP_BF, out=torch.empty(M, device=dev)))
                b = ev(); b.record()
                evs[k] += [a, b, m]
            torch.cuda.synchronize()
            for k, (a, b, m, c, d, m2) in enumerate(evs):
                ta[it, k] = (a.elapsed_time(b) + c.elapsed_time(d)) * 1e3
                if k == 0:
                    pa[it] = [a.elapsed_time(m) * 1e3, m.elapsed_time(b) * 1e3, c.elapsed_time(m2) * 1e3,
                              m2.elapsed_time(d) * 1e3]
            # adjoint
            evs = []
            sends = []
            for r, y in zip(ranks, yTs):
                a = ev(); a.record()
                r.phase(csd.DP_BA, inp=y)
                s = r.send_buffer(1)
                b = ev(); b.record()
                evs.append([a, b]); sends.append(s)
            recvs = csd.emulated_exchange(sends)
            for k, (r, buf) in enumerate(zip(ranks, recvs)):
                a = ev(); a.record()
                r.copy(1, False, buf)
                r.phase(csd.DP_C, out=torch.empty(r.nxc, device=dev))
                b = ev(); b.record()
                evs[k] += [a, b]
            torch.cuda.synchronize()
            for k, (a, b, c, d) in enumerate(evs):
                tt[it, k] = (a.elapsed_time(b) + c.elapsed_time(d)) * 1e3
        wa = float(np.max(np.median(ta, axis=0)))
        wt = float(np.max(np.median(tt, axis=0)))
        # the same per-rank halves replayed from CUDA graphs (dist.DistGraphs)
        graphs = [csd.DistGraphs(r) for r in ranks]
        ga = np.zeros((REPS, G)); gt = np.zeros((REPS, G))
        for it in range(REPS):
            for k, gr in enumerate(graphs):
                e = [ev() for _ in range(4)]
                e[0].record(); gr.pre_apply.replay(); e[1].record()
                e[2].record(); gr.post_apply.replay(); e[3].record()
                f = [ev() for _ in range(4)]
                f[0].record(); gr.pre_adjoint.replay(); f[1].record()
                f[2].record(); gr.post_adjoint.replay(); f[3].record()
                torch.cuda.synchronize()
                ga[it, k] = (e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3])) * 1e3
                gt[it, k] = (f[0].elapsed_time(f[1]) + f[2].elapsed_time(f[3])) * 1e3
        gwa = float(np.max(np.median(ga, axis=0)))
        gwt = float(np.max(np.median(gt, axis=0)))
        del graphs
        nv = sent / 900e9 * 1e6
        row = dict(N=N, G=G, single_apply_us=round(med(t1a), 1), single_adjoint_us=round(med(t1t), 1),
                   rank_apply_us=round(wa, 1), rank_adjoint_us=round(wt, 1),
                   rank_apply_graph_us=round(gwa, 1), rank_adjoint_graph_us=round(gwt, 1), a2a_bytes_per_rank=int(sent),
                   a2a_nvlink_us=round(nv, 1),
                   rank0_apply_A_pack_unpack_BF_us=[round(float(v), 1) for v in np.median(pa, axis=0)])
        rows_out.append(row)
        print(json.dumps(row), flush=True)
        del ranks, xcs, yTs
        torch.cuda.empty_cache()
