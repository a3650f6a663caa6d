"""Profiling driver: one full-size recovery of config PROF_CFG (no timing)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs, __graft_entry__
__graft_entry__.build()
import paper_1509_03979_b200 as cs
cid = int(os.environ.get("PROF_CFG", "5"))
prec = os.environ.get("PROF_PREC", "fp32")
cfg = cs_inputs.CONFIGS[cid]
B = int(os.environ.get("PROF_B", "1")) if cfg.batch > 1 else 1
td = torch.float32 if prec == "fp32" else torch.float64
dev = torch.device("cuda:0")
probs = cs_inputs.make_batch(cfg, count=B)
bits = torch.from_numpy(np.stack([p.sign_bits.view(np.int32) for p in probs])).to(dev)
rows = torch.from_numpy(np.stack([p.rows for p in probs]).astype(np.int32)).to(dev)
S = torch.from_numpy(np.stack([p.s for p in probs])).to(dev, td)
E = torch.from_numpy(np.stack([p.noise for p in probs])).to(dev, td)
A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=B)
Y = (cs.cs_operator_apply(A, S) + E).to(torch.float32).to(td)
X = cs.cs_operator_adjoint(A, Y)
r = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6 if prec == "fp32" else 1e-12)
torch.cuda.synchronize()
print(r.reports()[:2])
