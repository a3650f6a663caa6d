"""Per-phase time split of one Tier L recovery (GridCtx::mark accumulators)."""
import os, sys
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
S = torch.from_numpy(p.s[None]).to(dev, torch.float32)
Y = (cs.cs_operator_apply(A, S) + torch.from_numpy(p.noise[None]).to(dev, torch.float32))
ws = cs.Workspace()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
r = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6, workspace=ws)
ev0.record(); r = cs.cs_recover_batched(A, cfg.alg, Y, cfg.K, 1e-6, workspace=ws); ev1.record()
torch.cuda.synchronize()
tot = ev0.elapsed_time(ev1)
raw = ws.buf.cpu().numpy()
# ptime = ts area + 8 slots; locate the ts area: search for the accumulator block (values < 1e12 ns)
names = ["between sandwiches", "H pass A", "H pass B", "H pass C", "RES pass A", "RES pass B", "RES pass C+sum", "SP detection top-K", "CG setup", "OMPR(1) swap"]
rep = r.reports()[0]
print("total ms", tot, "outer", rep["outer_iters"], "cg", rep["cg_iters_total"], "applies", rep["applies"])
off = cs.load_library().cs_diag_phase_offset(cs.ALGS[cfg.alg], cfg.N, cfg.M, cfg.K, 0, 0)
acc = raw[off:off + 8 * 24].view(np.uint64)
# slots 10-14: pass-B item phases of H, only with CS_NVCC_EXTRA=-DCS_DIAG_PASSB
names += ["passB load+stage", "passB fwd FFT", "passB middle", "passB inv FFT", "passB twiddle+store",
          "CG x/r update", "CG rr reduction",  # 15-16: -DCS_DIAG_CG
          "set_input_support", "b gather", "CG loop exit", "cg_iterate entry"]  # 17-20: -DCS_DIAG_GLUE
print({n: round(float(v) / 1e6, 3) for n, v in zip(names, acc) if v}, "ms (block 0)")
