import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import __graft_entry__ as g; g.build()
import paper_1509_03979_b200 as cs
from paper_1509_03979_b200 import dist as csd
dev = torch.device("cuda:0")
for e in [16, 20, 24]:
    N = 1 << e; M = N // 4
    rng = np.random.default_rng(e)
    sign = rng.integers(0, 2**32, size=(1, N // 32), dtype=np.uint64).astype(np.uint32)
    rows = np.sort(rng.choice(N, size=M, replace=False)).astype(np.int32)[None]
    A = cs.Operator(N, M, torch.from_numpy(sign.view(np.int32)).to(dev), torch.from_numpy(rows).to(dev))
    for G in [1, 8]:
        r = csd.DistOperator(A, csd.dist_plan(N, G), 0)
        x = torch.randn(N, device=dev); w = torch.randn(M, device=dev)
        xc = r.scatter_x(x); yT = r.scatter_y(w)
        out = {}
        for name, fn in [("XS", lambda: r.scatter_x(x)), ("YT", lambda: r.scatter_y(w)),
                         ("A", lambda: r.phase(csd.DP_A, inp=xc)), ("BF", lambda: r.phase(csd.DP_BF, out=yT)),
                         ("BA", lambda: r.phase(csd.DP_BA, inp=yT)), ("C", lambda: r.phase(csd.DP_C, out=xc))]:
            ts = []
            for _ in range(20):
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
            out[name] = round(float(np.median(ts)), 1)
        print(e, G, out, flush=True)

# host time per phase call (no synchronization: the launch path alone), and one rank's apply
# (A, pack, unpack, BF) captured in a CUDA graph vs issued eagerly
import time
for e in [20, 24]:
    N = 1 << e; M = N // 4
    rng = np.random.default_rng(e)
    sign = rng.integers(0, 2**32, size=(1, N // 32), dtype=np.uint64).astype(np.uint32)
    rows = np.sort(rng.choice(N, size=M, replace=False)).astype(np.int32)[None]
    A = cs.Operator(N, M, torch.from_numpy(sign.view(np.int32)).to(dev), torch.from_numpy(rows).to(dev))
    for G in [1, 8]:
        r = csd.DistOperator(A, csd.dist_plan(N, G), 0)
        x = torch.randn(N, device=dev)
        xc = r.scatter_x(x)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            r.phase(csd.DP_XS, inp=x, out=xc)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        host_us = (t1 - t0) / 50 * 1e6
        sbuf, _, _ = r.send_buffer(0)
        rbuf = torch.zeros(sum(r.seg[(0, False)][2]), device=dev)
        yT = torch.empty(M, device=dev)

        def one():
            r.phase(csd.DP_A, inp=xc)
            r.copy(0, True, sbuf)
            r.copy(0, False, rbuf)
            r.phase(csd.DP_BF, out=yT)
        one(); torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                one()
        torch.cuda.synchronize()
        res = {}
        for name, fn in [("eager", one), ("graph", gr.replay)]:
            ts = []
            for _ in range(20):
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
            res[name] = round(float(np.median(ts)), 1)
        print(e, G, f"host us per phase call {host_us:.1f}", "rank apply", res, flush=True)
