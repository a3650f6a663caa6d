import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import __graft_entry__ as g; g.build()
import paper_1509_03979_b200 as cs, cs_inputs
alg = sys.argv[1]; N = int(sys.argv[2]); K = int(sys.argv[3]); prec = sys.argv[4]
cfg = cs_inputs.Config(80, alg, N, N // 4, K, "gauss", 0.0)
p = cs_inputs.make_problem(cfg)
dev = torch.device("cuda:0")
A = cs.Operator(N, N // 4, torch.from_numpy(p.sign_bits.view(np.int32)[None]).to(dev), torch.from_numpy(p.rows[None]).to(dev), batch=1)
td = torch.float32 if prec == "f32" else torch.float64
S = torch.from_numpy(p.s[None]).to(dev, td)
Y = cs.cs_operator_apply(A, S)
r = cs.cs_recover_batched(A, alg, Y, K, 1e-6 if prec == "f32" else 1e-12)
torch.cuda.synchronize()
print(alg, N, K, prec, "ok", r.reports()[0])
