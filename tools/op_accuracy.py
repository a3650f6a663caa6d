"""fp32 operator accuracy against the fp64 path (which matches the oracle to ~1e-13):
relative l2 and max-abs errors of apply / adjoint at several N (diagnostic)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs, __graft_entry__
__graft_entry__.build()
import paper_1509_03979_b200 as cs
dev = torch.device("cuda:0")
for l2n in [int(v) for v in os.environ.get("LOG2N", "14 16 20 24").split()]:
    N = 1 << l2n
    M = N // 4
    cfg = cs_inputs.Config(77, "sp", N, M, 8, "gauss", 0.0)
    p = cs_inputs.make_problem(cfg)
    bits = torch.from_numpy(p.sign_bits.view(np.int32)[None]).to(dev)
    rows = torch.from_numpy(p.rows[None].astype(np.int32)).to(dev)
    A = cs.Operator(N, M, bits, rows, batch=1)
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn((1, N), device=dev, dtype=torch.float64, generator=g)
    w = torch.randn((1, M), device=dev, dtype=torch.float64, generator=g)
    y64, y32 = cs.cs_operator_apply(A, x), cs.cs_operator_apply(A, x.float()).double()
    a64, a32 = cs.cs_operator_adjoint(A, w), cs.cs_operator_adjoint(A, w.float()).double()
    ey = ((y32 - y64).norm() / y64.norm()).item()
    ea = ((a32 - a64).norm() / a64.norm()).item()
    print(f"N=2^{l2n}: apply rel {ey:.3e}  adjoint rel {ea:.3e}", flush=True)
