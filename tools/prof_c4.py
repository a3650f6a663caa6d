"""Profiling driver (not a benchmark): build a config-4 batch and run the batched
apply, adjoint and one recover — small enough for `ncu --set full`."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs  # noqa: E402
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_1509_03979_b200 as cs  # noqa: E402

cid = int(os.environ.get("PROF_CFG", "4"))
B = int(os.environ.get("PROF_B", "1184"))
prec = os.environ.get("PROF_PREC", "fp32")
cfg = cs_inputs.CONFIGS[cid]
B = min(B, cfg.batch)
td = torch.float32 if prec == "fp32" else torch.float64
dev = torch.device("cuda:0")
probs = cs_inputs.make_batch(cfg, count=B)
bits = torch.from_numpy(np.stack([p.sign_bits.view(np.int32) for p in probs])).to(dev)
rows = torch.from_numpy(np.stack([p.rows for p in probs]).astype(np.int32)).to(dev)
S = torch.from_numpy(np.stack([p.s for p in probs])).to(dev, td)
A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=B)
Y = cs.cs_operator_apply(A, S)
X = cs.cs_operator_adjoint(A, Y)
r = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6 if prec == "fp32" else 1e-12)
torch.cuda.synchronize()
print(r.reports()[:2])
