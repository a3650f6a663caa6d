"""Diagnose c4 problems whose fp32 GPU support differs from the planted one."""
import sys, os
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import __graft_entry__ as g
g.build()
import paper_1509_03979_b200 as cs
import cs_inputs, oracle
from gpu_helpers import to_dev, measured, oracle_results, compare
cfg = cs_inputs.CONFIGS[4]
probs = cs_inputs.make_batch(cfg)
ys = measured(probs)
dev = torch.device("cuda:0")
bits, rows = to_dev(probs, dev)
A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=len(probs))
out = {}
for dt, tol in [("float32", 1e-6), ("float64", 1e-12)]:
    r = cs.cs_recover_batched(A, "sp", torch.from_numpy(ys).to(dev, getattr(torch, dt)), cfg.K, tol)
    torch.cuda.synchronize()
    out[dt] = (r.support.cpu().numpy(), r.values.cpu().numpy().astype(np.float64), r.reports())
planted = np.stack([p.support for p in probs])
s32 = out["float32"][0]; s64 = out["float64"][0]
miss32 = np.nonzero(~(s32 == planted).all(axis=1))[0]
miss64 = np.nonzero(~(s64 == planted).all(axis=1))[0]
print("miss fp32", miss32.size, "miss fp64", miss64.size, "fp32!=fp64", int((~(s32 == s64).all(axis=1)).sum()))
for i in miss32[:12]:
    ref = oracle_results([probs[i]], ys[i:i+1])[0]
    r32 = out["float32"][2][i]; r64 = out["float64"][2][i]
    print(i, "oracle==planted", np.array_equal(ref.support, planted[i]), "oracle outer", ref.outer_iters, getattr(ref, "termination", None),
          "| gpu32 outer", r32["outer_iters"], "term", r32["termination"], "res", r32["resid_norm"],
          "| gpu64==oracle", np.array_equal(np.sort(s64[i]), ref.support), "outer", r64["outer_iters"], "term", r64["termination"],
          "| symdiff32-or", np.setxor1d(s32[i], ref.support))
# margins: min |x_S| / ||x|| of the fp32 result, misses vs the whole batch
v32 = out["float32"][1]
rel = np.min(np.abs(v32), axis=1) / np.linalg.norm(v32, axis=1)
t32 = out["float32"][2]["termination"]
o32 = out["float32"][2]["outer_iters"]
print("miss min|x|/||x||:", np.round(rel[miss32], 9).tolist())
print("miss term:", t32[miss32].tolist(), "outer:", o32[miss32].tolist())
for thr in [1e-4, 3e-5, 1e-5, 3e-6, 1e-6]:
    fl = rel < thr
    print(f"flag min|x|/||x|| < {thr:g}: {int(fl.sum())} problems, misses caught {int(fl[miss32].sum())}/{miss32.size}")
print("term counts all:", np.bincount(t32).tolist(), "misses:", np.bincount(t32[miss32], minlength=5).tolist())
