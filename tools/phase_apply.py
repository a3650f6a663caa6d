"""Phase split of the Tier L apply at N = 2^24 (k_l_apply's %globaltimer stamps of block 0,
instance 0: input reorder, pass A, pass B, output permute).  Diagnostics, not a benchmark."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs, __graft_entry__
__graft_entry__.build()
import paper_1509_03979_b200 as cs
N = int(os.environ.get("PA_N", str(1 << 24)))
M = N // 4
dev = torch.device("cuda:0")
g = np.random.default_rng(1)
bits = torch.from_numpy(cs_inputs.pack_sign_bits(g.integers(0, 2, N).astype(bool)).view(np.int32)[None]).to(dev)
rows = torch.from_numpy(np.sort(g.choice(N, M, replace=False)).astype(np.int32)[None]).to(dev)
A = cs.Operator(N, M, bits, rows, batch=1)
X = torch.randn((1, N), device=dev)
for _ in range(3):
    Y = cs.cs_operator_apply(A, X)
torch.cuda.synchronize()
ws, nb = A.ws(torch.float32)
off = cs.load_library().cs_diag_phase_offset(-1, N, M, 8, 0, 0)
ts = ws.view(torch.uint8)[off:off + 40].cpu().numpy().view(np.uint64).astype(np.int64)
d = np.diff(ts) / 1e3
print(f"N=2^{int(np.log2(N))} apply phases (us): reorder {d[0]:.1f}, pass A {d[1]:.1f}, pass B {d[2]:.1f}, permute {d[3]:.1f}, total {(ts[4]-ts[0])/1e3:.1f}")
