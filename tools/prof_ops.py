"""Standalone operator and top-K kernels: CUDA-event timing (no profiler) and achieved GB/s
against MEASURED_PEAKS.json, for the kernels the recovery fuses (per-kernel HBM
evidence for the operator and top-K).  Shapes: the c4 batch (4096 x N = 2^14, Tier S), one
c5-size vector (N = 2^24, Tier L), the grid top-K at c5's detection (2^24 keys -> 65536) and
the CTA top-K at c4's (2^14 keys -> 256).  Under ncu (PROF_ONCE=1) each kernel runs once.

Algorithmic bytes per launch:
  apply   B (4N + 4M + 3N/32 metadata) — x read, y written, sign / row-mask / prefix words
  adjoint the same (y read, x written)
  top-K   4n (keys read once) + n/8 (bit mask written)
"""
import ctypes
import json
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

ONCE = os.environ.get("PROF_ONCE") == "1"
dev = torch.device("cuda:0")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6542.4)


def timed(fn, reps=10):
    if ONCE:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


rows_out = []


def op_case(name, N, B):
    M = N // 4
    g = np.random.default_rng(N)
    bits = torch.from_numpy(cs_inputs.pack_sign_bits(g.integers(0, 2, (B, N)).astype(bool).reshape(-1))
                            .view(np.int32).reshape(B, -1)).to(dev)
    rows = torch.from_numpy(np.stack([np.sort(g.choice(N, M, replace=False)) for _ in range(B)]).astype(np.int32)).to(dev)
    A = cs.Operator(N, M, bits, rows, batch=B)
    X = torch.randn((B, N), device=dev)
    Y = torch.empty((B, M), device=dev)
    Xo = torch.empty((B, N), device=dev)
    nbytes = B * (4 * N + 4 * M + 3 * N // 32 * 4 // 4 * 4 // 4)
    nbytes = B * (4 * N + 4 * M + 3 * (N // 32) * 4)
    ta = timed(lambda: cs.cs_operator_apply(A, X, out=Y))
    tj = timed(lambda: cs.cs_operator_adjoint(A, Y, out=Xo))
    rows_out.append((f"{name} apply", B, N, ta, nbytes))
    rows_out.append((f"{name} adjoint", B, N, tj, nbytes))


def topk_case(name, n, K, grid):
    lib = cs.load_library()
    v = torch.randn(n, device=dev)
    out = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if grid:
        ws = torch.empty(int(lib.cs_diag_topk_grid_ws_bytes()), dtype=torch.uint8, device=dev)
        fn = lambda: lib.cs_diag_topk_grid(ctypes.c_void_p(v.data_ptr()), n, K, 0, ctypes.c_void_p(out.data_ptr()),
                                           ctypes.c_void_p(ws.data_ptr()), ws.numel(), st)
    else:
        fn = lambda: lib.cs_diag_topk(ctypes.c_void_p(v.data_ptr()), n, K, 0, 0, ctypes.c_void_p(out.data_ptr()), st)
    t = timed(fn)
    rows_out.append((name, 1, n, t, 4 * n + n // 8))


op_case("c4 shape (Tier S)", 1 << 14, 4096)
op_case("c5 size (Tier L)", 1 << 24, 1)
topk_case("grid top-K 2^24 -> 65536 (c5 detection)", 1 << 24, 65536, True)
topk_case("CTA top-K 2^14 -> 256 (c4 detection, one CTA)", 1 << 14, 256, False)
if not ONCE:
    print("| kernel | batch | N | ms | algorithmic GB/s | fraction of HBM (%.0f GB/s, measured) |" % peak)
    print("|---|---|---|---|---|---|")
    for name, B, N, t, nb in rows_out:
        print(f"| {name} | {B} | 2^{int(np.log2(N))} | {t * 1e3:.4f} | {nb / t / 1e9:.1f} | {nb / t / 1e9 / peak:.3f} |")
