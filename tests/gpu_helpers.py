"""Shared setup for the -m gpu tests: seeded problems -> device tensors -> CUDA path."""
import numpy as np

import cs_inputs
import oracle


def to_dev(problems, dev):
    import torch
    bits = torch.from_numpy(np.stack([p.sign_bits.view(np.int32) for p in problems])).to(dev)
    rows = torch.from_numpy(np.stack([p.rows for p in problems]).astype(np.int32)).to(dev)
    return bits, rows


def perms_dev(problems, dev):
    """[B][N] int32 permutations of the Eq.(7) randomizer (R34), or None."""
    import torch
    if problems[0].perm is None:
        return None
    return torch.from_numpy(np.stack([p.perm for p in problems]).astype(np.int32)).to(dev)


def measured(problems):
    """y via the ORACLE operator, rounded to fp32 (R21)."""
    ys = []
    for p in problems:
        op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
        ys.append((op.apply(p.s) + p.noise).astype(np.float32))
    return np.stack(ys)


def oracle_results(problems, ys, tol=1e-10, **kw):
    out = []
    for p, y in zip(problems, ys):
        op = oracle.SrmOperator(p.N, p.sign_bits, p.rows, p.perm, p.psi, p.transform)
        out.append(oracle.recover(p.alg, op, y.astype(np.float64), p.K, tol=tol, **kw))
    return out


def dense_from(N, supp, vals):
    s = np.zeros(N)
    s[supp] = vals
    return s


def compare(problems, refs, supp, vals, rtol=1e-4):
    """BASELINE.json parity bar: identical supports, ||s_gpu - s_oracle|| / ||s_oracle|| <= 1e-4."""
    bad = []
    worst = 0.0
    for b, (p, ref) in enumerate(zip(problems, refs)):
        sg = np.sort(supp[b])
        if not np.array_equal(sg, ref.support):
            bad.append((b, "support", int(np.setxor1d(sg, ref.support).size)))
            continue
        s_gpu = dense_from(p.N, supp[b], vals[b].astype(np.float64))
        rel = np.linalg.norm(s_gpu - ref.s_hat) / max(np.linalg.norm(ref.s_hat), 1e-300)
        worst = max(worst, rel)
        if rel > rtol:
            bad.append((b, "coef", rel))
    return bad, worst


def compare_fp32_floor(problems, refs, supp, vals, rtol=1e-4, floor=1e-5):
    """compare() for fp32 results on problems where a support index can sit below fp32
    resolution: a support mismatch is accepted only when every index in
    the symmetric difference carries |s_oracle_j| <= floor * ||s_oracle|| (a coefficient
    the fp32 sandwich cannot resolve) and the dense coefficients still agree to rtol."""
    bad = []
    for b, (p, ref) in enumerate(zip(problems, refs)):
        sg = np.sort(supp[b])
        s_gpu = dense_from(p.N, supp[b], vals[b].astype(np.float64))
        nrm = max(np.linalg.norm(ref.s_hat), 1e-300)
        rel = np.linalg.norm(s_gpu - ref.s_hat) / nrm
        if not np.array_equal(sg, ref.support):
            diff = np.setxor1d(sg, ref.support)
            if np.max(np.abs(ref.s_hat[diff])) > floor * nrm:
                bad.append((b, "support", int(diff.size)))
                continue
        if rel > rtol:
            bad.append((b, "coef", rel))
    return bad
