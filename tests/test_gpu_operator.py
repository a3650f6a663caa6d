"""GPU parity of the operator A = P.DCT-II.diag(sigma) and its adjoint (cs_operator_apply /
cs_operator_adjoint) against the fp64 oracle, both tiers, fp32 and fp64, through the C ABI."""
import numpy as np
import pytest

import cs_inputs
import oracle
from gpu_helpers import to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def _setup(N, M, batch, seed=0):
    cfg = cs_inputs.Config(70 + seed, "sp", N, M, max(1, M // 8), "gauss", 0.0)
    return [cs_inputs.make_problem(cfg, b=b) for b in range(batch)]


# Tier S: N <= 16384 (one CTA per vector); Tier L: four-step cooperative grid.
SIZES = [(8, 4, 3), (16, 8, 2), (32, 8, 2), (64, 16, 3), (256, 64, 2), (1024, 256, 2), (4096, 1024, 2),
         (16384, 4096, 3), (32768, 8192, 1), (65536, 16384, 2), (1 << 18, 1 << 16, 1), (1 << 20, 1 << 18, 1),
         # the full-size grid-tier shapes: c5's N = 2^24 (pass tiles of 4096 points) and beyond
         (1 << 22, 1 << 20, 1), (1 << 24, 1 << 22, 1), (1 << 25, 1 << 23, 1)]


@pytest.mark.parametrize("N,M,batch", SIZES)
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_apply_adjoint_match_oracle(cs, N, M, batch, dtype):
    dev = torch.device("cuda:0")
    probs = _setup(N, M, batch)
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(N, M, bits, rows, batch=batch)
    g = np.random.default_rng(N + batch)
    X = g.standard_normal((batch, N))
    W = g.standard_normal((batch, M))
    td = getattr(torch, dtype)
    Yg = cs.cs_operator_apply(A, torch.from_numpy(X).to(dev, td)).cpu().numpy().astype(np.float64)
    Xg = cs.cs_operator_adjoint(A, torch.from_numpy(W).to(dev, td)).cpu().numpy().astype(np.float64)
    tol = 2e-6 if dtype == "float32" else 1e-13
    for b, p in enumerate(probs):
        op = oracle.SrmOperator(N, p.sign_bits, p.rows)
        y_ref = op.apply(X[b])
        x_ref = op.adjoint(W[b])
        ey = np.linalg.norm(Yg[b] - y_ref) / np.linalg.norm(y_ref)
        ex = np.linalg.norm(Xg[b] - x_ref) / np.linalg.norm(x_ref)
        assert ey <= tol, (b, ey)
        assert ex <= tol, (b, ex)
        # element-wise: worst entry relative to the vector scale
        assert np.max(np.abs(Yg[b] - y_ref)) <= 10 * tol * np.linalg.norm(y_ref) / np.sqrt(M) * np.sqrt(np.log2(N) + 1) + 1e-300


@pytest.mark.parametrize("N,M", [(4096, 1024), (1 << 16, 1 << 14)])
def test_adjoint_identity_and_rows_orthonormal(cs, N, M):
    dev = torch.device("cuda:0")
    probs = _setup(N, M, 1, seed=3)
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(N, M, bits, rows)
    g = np.random.default_rng(1)
    x = torch.from_numpy(g.standard_normal((1, N))).to(dev, torch.float64)
    w = torch.from_numpy(g.standard_normal((1, M))).to(dev, torch.float64)
    lhs = float((cs.cs_operator_apply(A, x) * w).sum())
    rhs = float((x * cs.cs_operator_adjoint(A, w)).sum())
    assert abs(lhs - rhs) <= 1e-11 * float(x.norm() * w.norm())
    # A A^T = I on the selected rows
    aat = cs.cs_operator_apply(A, cs.cs_operator_adjoint(A, w))
    assert float((aat - w).norm()) <= 1e-12 * float(w.norm())


def test_zero_and_impulse(cs):
    dev = torch.device("cuda:0")
    N, M = 2048, 512
    probs = _setup(N, M, 1, seed=5)
    bits, rows = to_dev(probs, dev)
    A = cs.Operator(N, M, bits, rows)
    z = torch.zeros((1, N), device=dev)
    assert float(cs.cs_operator_apply(A, z).abs().max()) == 0.0
    assert float(cs.cs_operator_adjoint(A, torch.zeros((1, M), device=dev)).abs().max()) == 0.0
    # column j of A: A e_j = sigma_j C_N[rows, j]
    op = oracle.SrmOperator(N, probs[0].sign_bits, probs[0].rows)
    for j in [0, 1, N // 2, N - 1]:
        e = torch.zeros((1, N), device=dev, dtype=torch.float64)
        e[0, j] = 1
        ej = np.zeros(N)
        ej[j] = 1
        np.testing.assert_allclose(cs.cs_operator_apply(A, e).cpu().numpy()[0], op.apply(ej), atol=1e-14)


def test_bad_rows_rejected(cs):
    dev = torch.device("cuda:0")
    N, M = 64, 4
    bits = torch.zeros((1, 2), dtype=torch.int32, device=dev)
    for rows in ([0, 5, 5, 9], [3, 2, 7, 9], [0, 1, 2, 64], [-1, 1, 2, 3]):
        with pytest.raises(cs.CsError) as ei:
            cs.Operator(N, M, bits, torch.tensor([rows], dtype=torch.int32, device=dev))
        assert ei.value.status == 1


def test_bad_sizes_rejected(cs):
    dev = torch.device("cuda:0")
    bits = torch.zeros((1, 4), dtype=torch.int32, device=dev)
    rows = torch.arange(8, dtype=torch.int32, device=dev)[None]
    with pytest.raises(cs.CsError) as ei:
        cs.Operator(100, 8, bits, rows)
    assert ei.value.status == 2
    with pytest.raises(cs.CsError) as ei:
        cs.Operator(4, 2, bits, rows[:, :2])
    assert ei.value.status == 2
