"""The paper's precision study (Tables II-IV; SNR remarks P:627-632) on the B200
path — SURVEY §8f NEXT-2.

Paper regime: M = N/4, K = M/4, s ~ p N(0, 1) (Bernoulli-Gaussian, p = K/N),
y = A s + eta with sigma_eta = 0.01; CG-OMP, CG-OMPR and CG-SP at CG precision
xi in {"exact", 1e-10, 1e-5}.  Readings (R7/R8): xi is relative to ||b||; "exact"
is xi = 1e-13 with the fp64 path; 1e-10 also runs in fp64 (below the fp32 floor); 1e-5 runs
in fp32 (the headline precision) and fp64.  A is this build's operator (BASELINE.json:
P.DCT-II.diag(sigma), Psi = I), not the paper's D.F.R with Psi = DCT — the numbers are
the shape of the paper's tables on this hardware, not a reproduction of its Matlab timings.

SNR = 20 log10(||s|| / ||s - s_hat||) (R30).  Output: a markdown table.

  python tools/precision_study.py [--max-log2n 24] [--algs omp,ompr,sp] [--out FILE]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cs_inputs  # noqa: E402
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_1509_03979_b200 as cs  # noqa: E402

XI = [("exact (1e-13, fp64)", 1e-13, torch.float64), ("1e-10 (fp64)", 1e-10, torch.float64),
      ("1e-5 (fp64)", 1e-5, torch.float64), ("1e-5 (fp32)", 1e-5, torch.float32)]
LIMITS = {"omp": 16, "ompr": 18, "sp": 24}   # largest log2 N per algorithm by default


def problem(N, seed):
    """Eq.(13): each entry nonzero with probability p = K/N, N(0,1) values; noise 0.01."""
    M, K = N // 4, N // 16
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([1509, N, seed])))
    sign_bits = cs_inputs.pack_sign_bits(g.integers(0, 2, N).astype(bool))
    rows = np.sort(g.choice(N, M, replace=False)).astype(np.int32)
    s = np.where(g.random(N) < K / N, g.standard_normal(N), 0.0)
    noise = 0.01 * g.standard_normal(M)
    return M, K, sign_bits, rows, s, noise


def run(alg, N, seed=0):
    dev = torch.device("cuda:0")
    M, K, sign_bits, rows, s, noise = problem(N, seed)
    bits = torch.from_numpy(sign_bits.view(np.int32)[None]).to(dev)
    rws = torch.from_numpy(rows[None]).to(dev)
    A = cs.Operator(N, M, bits, rws, batch=1)
    s64 = torch.from_numpy(s[None]).to(dev, torch.float64)
    y64 = cs.cs_operator_apply(A, s64) + torch.from_numpy(noise[None]).to(dev)
    y32 = y64.to(torch.float32)
    out = []
    for name, xi, td in XI:
        Y = y32.to(td)          # the same fp32-rounded measurements for every run (R21)
        ws = cs.Workspace()
        cs.cs_recover_batched(A, alg, Y, K, xi, workspace=ws)   # warm-up (workspace, tables)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = cs.cs_recover_batched(A, alg, Y, K, xi, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        rep = r.reports()[0]
        sh = np.zeros(N)
        sh[r.support.cpu().numpy()[0]] = r.values.cpu().numpy()[0].astype(np.float64)
        snr = 20 * np.log10(np.linalg.norm(s) / np.linalg.norm(s - sh))
        out.append((name, e0.elapsed_time(e1) / 1e3, int(rep["cg_iters_total"]), int(rep["outer_iters"]), snr))
    return M, K, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2n", type=int, default=11)
    ap.add_argument("--max-log2n", type=int, default=24)
    ap.add_argument("--algs", default="omp,ompr,sp")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    lines = ["| alg | N | M | K | xi | time (s) | CG iters | outer | SNR (dB) | dSNR vs exact (dB) |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for alg in a.algs.split(","):
        for l2 in range(a.min_log2n, min(a.max_log2n, LIMITS[alg]) + 1):
            t0 = time.time()
            M, K, res = run(alg, 1 << l2)
            base = res[0][4]
            for name, t, cg, outer, snr in res:
                lines.append(f"| {alg} | 2^{l2} | {M} | {K} | {name} | {t:.4f} | {cg} | {outer} | {snr:.3f} | {snr - base:+.4f} |")
            print(lines[-1], f"[{time.time() - t0:.1f}s wall]", flush=True)
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
