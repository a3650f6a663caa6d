import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1509_03979_b200 as cs
from paper_1509_03979_b200 import dist as csd
dev = torch.device("cuda:0")
for e in [16, 24]:
    N = 1 << e; M = N // 4
    rng = np.random.default_rng(e)
    sign = rng.integers(0, 2**32, size=(1, N // 32), dtype=np.uint64).astype(np.uint32)
    rows = np.sort(rng.choice(N, size=M, replace=False)).astype(np.int32)[None]
    A = cs.Operator(N, M, torch.from_numpy(sign.view(np.int32)).to(dev), torch.from_numpy(rows).to(dev))
    r = csd.DistOperator(A, csd.dist_plan(N, 8), 0)
    x = torch.randn(N, device=dev); w = torch.randn(M, device=dev)
    xc = r.scatter_x(x); yT = r.scatter_y(w)
    for _ in range(2):
        r.scatter_x(x); r.phase(csd.DP_A, inp=xc); r.phase(csd.DP_BF, out=yT); r.phase(csd.DP_BA, inp=yT); r.phase(csd.DP_C, out=xc)
    torch.cuda.synchronize()
