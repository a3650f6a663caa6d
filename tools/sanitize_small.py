"""Small recoveries on every tier / algorithm / precision, for compute-sanitizer."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs, __graft_entry__
__graft_entry__.build()
import paper_1509_03979_b200 as cs
dev = torch.device("cuda:0")
cases = [cs_inputs.CONFIGS[1].scaled(4), cs_inputs.CONFIGS[4].scaled(8, batch=3),
         cs_inputs.Config(70, "ompr", 4096, 1024, 32, "pm1", 0.0),
         cs_inputs.CONFIGS[2].scaled(2), cs_inputs.Config(71, "ompr", 1 << 16, 1 << 14, 64, "pm1", 0.0),
         cs_inputs.Config(72, "omp", 1 << 15, 1 << 13, 16, "gauss", 0.0)]
for cfg in cases:
    B = min(cfg.batch, 3)
    probs = cs_inputs.make_batch(cfg, count=B)
    bits = torch.from_numpy(np.stack([p.sign_bits.view(np.int32) for p in probs])).to(dev)
    rows = torch.from_numpy(np.stack([p.rows for p in probs]).astype(np.int32)).to(dev)
    for td in (torch.float32, torch.float64):
        S = torch.from_numpy(np.stack([p.s for p in probs])).to(dev, td)
        A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=B)
        Y = cs.cs_operator_apply(A, S)
        X = cs.cs_operator_adjoint(A, Y)
        r = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6 if td == torch.float32 else 1e-12)
        torch.cuda.synchronize()
        print(cfg.alg, cfg.N, td, r.reports()["termination"])
print("sanitize ok")
