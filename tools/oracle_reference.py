"""Full-size oracle references for the configs the oracle cannot finish inside a test.

Runs the fp64 oracle (`oracle/` only — never the CUDA path) on BASELINE.json config 3
(OMPR(1), N = 2^20) and config 5 (SP, N = 2^24) at full size, with the same seeded
inputs as the GPU tests (cs_inputs, trial 0, problem 0; y formed with the ORACLE
operator and rounded to fp32, R21), and stores the answer under
tests/golden/ for tests/test_gpu_full.py:

  oracle_c<k>.npz: support (int32, ascending), x (float64, values on the support),
                   outer_iters, cg_iters, termination, resid_norm, y_sha (sha256 of the
                   fp32 y bytes, so a test can prove it feeds the same input), tol.

Usage: python tools/oracle_reference.py 3 5     (c3 ~10-15 min, c5 ~7 min on one core)
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import cs_inputs  # noqa: E402
import oracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def y_of(p):
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    return op, (op.apply(p.s) + p.noise).astype(np.float32)


def y_sha(y32: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(y32, dtype=np.float32).tobytes()).hexdigest()


def run(cid: int, tol: float = 1e-10) -> str:
    cfg = cs_inputs.CONFIGS[cid]
    p = cs_inputs.make_problem(cfg, 0, 0)
    op, y32 = y_of(p)
    t0 = time.time()
    res = oracle.recover(p.alg, op, y32.astype(np.float64), p.K, tol=tol)
    dt = time.time() - t0
    out = os.path.join(GOLDEN, f"oracle_c{cid}.npz")
    np.savez_compressed(out, support=res.support.astype(np.int32), x=res.x.astype(np.float64),
                        outer_iters=res.outer_iters, cg_iters=res.cg_iters, termination=res.termination,
                        resid_norm=res.resid_norm, y_sha=y_sha(y32), tol=tol, seconds=dt,
                        resid_history=np.asarray(res.resid_history))
    print(f"c{cid}: {dt:.1f} s, outer {res.outer_iters}, cg {res.cg_iters}, term {res.termination}, "
          f"|S| {res.support.size}, planted overlap {np.intersect1d(res.support, p.support).size} -> {out}",
          flush=True)
    return out


if __name__ == "__main__":
    for a in sys.argv[1:] or ["3", "5"]:
        run(int(a))
