"""Test-side helpers: y = A s + eta via the ORACLE operator (never the CUDA path).

Per SURVEY §8c.7 #21 / DESIGN.md R21: y is generated in fp64, rounded to fp32,
and the same fp32 y (upcast) is fed to both the oracle and the GPU.
"""
import numpy as np

import cs_inputs
import oracle


def measure(p: cs_inputs.Problem):
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    y = op.apply(p.s) + p.noise
    y32 = y.astype(np.float32)
    return op, y32


def oracle_recover(p: cs_inputs.Problem, y32, tol=1e-10, **kw):
    op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
    return oracle.recover(p.alg, op, y32.astype(np.float64), p.K, tol=tol, **kw)
