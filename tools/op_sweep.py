"""Operator applies/sec and HBM GB/s of the batched apply / adjoint across N (BJ metric
"operator applies/sec; achieved HBM GB/s vs peak").  Batch B = max(1, 2^26 / N) so every
launch moves ~256 MB of x; CUDA-event timing of 10 launches after 3 warm-ups.

  python tools/op_sweep.py [--out profiles/r01/op_sweep.md]
"""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    dev = torch.device("cuda:0")
    lines = ["| N | batch | apply ms | applies/s | apply GB/s | adjoint ms | adjoint GB/s | tier |",
             "|---|---|---|---|---|---|---|---|"]
    for l2 in range(10, 25):
        N = 1 << l2
        M = N // 4
        B = max(1, (1 << 26) // N)
        cfg = cs_inputs.Config(79, "sp", N, M, 8, "gauss", 0.0)
        g = np.random.default_rng(l2)
        bits = torch.from_numpy(cs_inputs.pack_sign_bits(g.integers(0, 2, (B, N)).astype(bool).reshape(-1))
                                .view(np.int32).reshape(B, -1)).to(dev)
        rows = torch.from_numpy(np.stack([np.sort(g.choice(N, M, replace=False)) for _ in range(B)])
                                .astype(np.int32)).to(dev)
        A = cs.Operator(N, M, bits, rows, batch=B)
        X = torch.randn((B, N), device=dev)
        W = torch.randn((B, M), device=dev)
        res = []
        for fn, arg in ((cs.cs_operator_apply, X), (cs.cs_operator_adjoint, W)):
            for _ in range(3):
                fn(A, arg)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn(A, arg)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 10)
        nbytes = B * (4 * N + 4 * M + 3 * N // 8 + (4 * M if N > 16384 else 0))
        ms_f, ms_a = res
        lines.append(f"| 2^{l2} | {B} | {ms_f:.4f} | {B / ms_f * 1e3:.3g} | {nbytes / ms_f / 1e6:.0f} "
                     f"({nbytes / ms_f / 1e6 / peak:.2f}) | {ms_a:.4f} | {nbytes / ms_a / 1e6:.0f} "
                     f"({nbytes / ms_a / 1e6 / peak:.2f}) | {'CTA' if N <= 16384 else 'grid'} |")
        print(lines[-1], flush=True)
    txt = "\n".join(lines)
    if a.out:
        open(a.out, "w").write(f"HBM peak (MEASURED_PEAKS.json): {peak} GB/s\n\n" + txt + "\n")


if __name__ == "__main__":
    main()
