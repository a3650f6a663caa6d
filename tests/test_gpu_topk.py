"""Bit-exact parity of the CTA tier's top-K selection (b2) with the oracle's
definition (oracle.topk: the K largest |v|, ties to the lowest index, §8c.6), on
adversarial inputs: heavy ties at the boundary, exact zeros, K = n, denormals, values
that differ only in the last mantissa bits (the two-pass path's candidate resolution),
and sizes that overflow the candidate list (radix fallback).  Through the C ABI test
hook cs_diag_topk; both the two-pass path (mode 0) and the radix path (mode 1)."""
import ctypes

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cs():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as m
    return m


def gpu_topk(cs, v, K, mode):
    dev = torch.device("cuda:0")
    t = torch.from_numpy(v).to(dev)
    out = torch.zeros((v.size + 31) // 32, dtype=torch.int32, device=dev)
    prec = 1 if v.dtype == np.float64 else 0
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = cs.load_library().cs_diag_topk(ctypes.c_void_p(t.data_ptr()), v.size, K, prec, mode,
                                        ctypes.c_void_p(out.data_ptr()), st)
    assert rc == 0, cs.load_library().cs_last_error()
    torch.cuda.synchronize()
    bits = np.unpackbits(out.cpu().numpy().view(np.uint8), bitorder="little")[: v.size]
    return np.nonzero(bits)[0]


def cases():
    rng = np.random.default_rng(7)
    out = []
    for dt in (np.float32, np.float64):
        n = 16384
        out.append(("gauss", rng.standard_normal(n).astype(dt), 256))
        v = np.round(rng.standard_normal(n) * 4).astype(dt)          # integers: massive ties
        out.append(("integer-ties", v, 300))
        v = np.zeros(n, dt)
        v[rng.choice(n, 100, replace=False)] = 1.0                    # 100 ones, rest exact zeros
        out.append(("zeros-fill", v, 256))
        base = dt(1.2345)
        v = np.full(n, base, dtype=dt)
        v = v + (rng.integers(0, 8, n) * np.finfo(dt).eps).astype(dt)  # last-ulp differences
        out.append(("last-ulp", v, 777))
        out.append(("K=n", rng.standard_normal(513).astype(dt), 513))
        out.append(("tiny-n", np.array([3, -3, 1, 0, -1], dt), 2))
        v = (rng.standard_normal(n) * 1e-39).astype(dt)               # fp32 denormals
        out.append(("denormal", v, 100))
        v = np.abs(rng.standard_normal(5000)).astype(dt)
        v[::7] = v[0]                                                 # a tied value across the range
        out.append(("one-value-tied", v, 2000))
    return out


@pytest.mark.parametrize("mode", [0, 1])
def test_topk_matches_oracle_definition(cs, mode):
    for name, v, K in cases():
        got = gpu_topk(cs, v, K, mode)
        want = oracle.topk(np.abs(v.astype(np.float64)) if v.dtype == np.float64 else np.abs(v), K)
        assert np.array_equal(got, want), (name, v.dtype, mode, np.setxor1d(got, want)[:10])


# ---- the grid tier's radix top-K (detection at N >= 2^15: c2, c3, c5), full cooperative grid
def gpu_topk_grid(cs, v, K):
    lib = cs.load_library()
    dev = torch.device("cuda:0")
    t = torch.from_numpy(v).to(dev)
    out = torch.zeros((v.size + 31) // 32, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib.cs_diag_topk_grid_ws_bytes()), dtype=torch.uint8, device=dev)
    prec = 1 if v.dtype == np.float64 else 0
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = lib.cs_diag_topk_grid(ctypes.c_void_p(t.data_ptr()), v.size, K, prec, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(ws.data_ptr()), ws.numel(), st)
    assert rc == 0, lib.cs_last_error()
    torch.cuda.synchronize()
    bits = np.unpackbits(out.cpu().numpy().view(np.uint8), bitorder="little")[: v.size]
    return np.nonzero(bits)[0]


def grid_cases():
    rng = np.random.default_rng(11)
    out = []
    for dt in (np.float32, np.float64):
        for n, K in [(1 << 16, 2048), (1 << 20, 8192), (1 << 24, 65536)]:
            out.append((f"gauss-{n}", rng.standard_normal(n).astype(dt), K))
        n = 1 << 20
        out.append(("integer-ties", np.round(rng.standard_normal(n) * 4).astype(dt), 9000))
        v = np.zeros(n, dt)
        v[rng.choice(n, 3000, replace=False)] = 1.0                   # fewer nonzeros than K
        out.append(("zeros-fill", v, 8192))
        v = np.full(n, dt(1.2345), dtype=dt) + (rng.integers(0, 8, n) * np.finfo(dt).eps).astype(dt)
        out.append(("last-ulp", v, 65536))
        v = (rng.standard_normal(1 << 16) * 1e-39).astype(dt)
        out.append(("denormal", v, 1000))
        out.append(("all-equal", np.full(1 << 18, dt(-2.5), dtype=dt), 12345))
        out.append(("K=n", rng.standard_normal(70000).astype(dt), 70000))
        v = np.abs(rng.standard_normal(1 << 24)).astype(dt)
        v[::3] = v[5]                                                 # one value tied across 2^24 / 3 slots
        out.append(("tied-2^24", v, 65536))
    return out


def test_grid_topk_matches_oracle_definition(cs):
    for name, v, K in grid_cases():
        got = gpu_topk_grid(cs, v, K)
        want = oracle.topk(np.abs(v.astype(np.float64)) if v.dtype == np.float64 else np.abs(v), K)
        assert np.array_equal(got, want), (name, v.dtype, np.setxor1d(got, want)[:10])
