"""Phase timing of the Tier L apply (diagnostic stamps in the workspace control block)."""
import os, sys, ctypes
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs, __graft_entry__
__graft_entry__.build()
import paper_1509_03979_b200 as cs
cid = int(os.environ.get("PROF_CFG", "5"))
cfg = cs_inputs.CONFIGS[cid]
dev = torch.device("cuda:0")
p = cs_inputs.make_problem(cfg)
bits = torch.from_numpy(p.sign_bits.view(np.int32)[None]).to(dev)
rows = torch.from_numpy(p.rows[None].astype(np.int32)).to(dev)
A = cs.Operator(cfg.N, cfg.M, bits, rows, batch=1)
X = torch.randn((1, cfg.N), device=dev)
for _ in range(3):
    Y = cs.cs_operator_apply(A, X)
torch.cuda.synchronize()
ws, nb = A.ws(torch.float32)
raw = ws.cpu().numpy()
# the ts area is the last 64*8 bytes before ctl_end; find it by scanning for the stamp pattern
# (layout offsets are not exported; read the last 2 KB and look for 5 increasing ~1.7e18 values)
tail = raw[-8192:].view(np.uint64)
cand = [i for i in range(len(tail) - 5) if 1e18 < tail[i] < 3e18 and all(tail[i + k] >= tail[i + k - 1] for k in range(1, 5))]
i = cand[0]
t = tail[i:i + 5].astype(np.int64)
print("phases (us): input", (t[1] - t[0]) / 1e3, "passA", (t[2] - t[1]) / 1e3, "passB", (t[3] - t[2]) / 1e3, "perm", (t[4] - t[3]) / 1e3)
