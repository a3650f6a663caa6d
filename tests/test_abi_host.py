"""Host-only checks of the C ABI (no GPU needed): the library loads, exports every
symbol include/cs.h declares, and host-side validation returns the documented codes."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    import paper_1509_03979_b200 as cs
    return cs.load_library()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_binding_declares_every_export():
    import paper_1509_03979_b200 as cs
    assert sorted(cs.EXPORTS) == declared_functions()


def test_status_strings_and_version(lib):
    assert lib.cs_status_string(0) == b"CS_OK"
    assert lib.cs_status_string(3) == b"CS_ERR_WORKSPACE"
    assert b"sm_100a" in lib.cs_version()


def test_meta_bytes_formula(lib):
    # N <= 16384: sign + natural mask/prefix + transposed mask/prefix (5 word arrays of
    # ceil(N/32)) + an M-entry int32 permutation per instance, 256-aligned, + 256 flag tail
    assert lib.cs_operator_meta_bytes(16384, 4096, 4096) == \
        ((4096 * (5 * 512 + 4096) * 4 + 255) // 256) * 256 + 256
    assert lib.cs_operator_meta_bytes(8, 4, 1) == 256 + 256
    # N > 16384 (Tier L only): sign + transposed mask/prefix + permutation
    N, M = 1 << 20, 1 << 18
    assert lib.cs_operator_meta_bytes(N, M, 1) == ((3 * (N // 32) * 4 + M * 4 + 255) // 256) * 256 + 256


def test_host_validation_codes(lib):
    import paper_1509_03979_b200 as cs
    n = ctypes.c_size_t()
    # N not a power of two / out of range -> UNSUPPORTED
    assert lib.cs_workspace_bytes(1, 100, 25, 4, 1, 0, None, ctypes.byref(n)) == 2
    assert lib.cs_workspace_bytes(1, 1 << 26, 1 << 24, 4, 1, 0, None, ctypes.byref(n)) == 2
    # bad K -> INVALID_ARG
    assert lib.cs_workspace_bytes(1, 1024, 256, 0, 1, 0, None, ctypes.byref(n)) == 1
    # null out pointer -> INVALID_ARG
    h = ctypes.c_void_p()
    assert lib.cs_operator_create(1024, 256, 1, None, None, None, 0, None, ctypes.byref(h)) == 1
    assert lib.cs_operator_create(1024, 2048, 1, None, None, None, 0, None, ctypes.byref(h)) == 1
    # workspace sizes: Tier S = B*2N*sizeof(T) (A^T y + the Psi = DCT scratch); Tier L
    # larger than the dense scratch
    assert lib.cs_workspace_bytes(1, 16384, 4096, 256, 4096, 0, None, ctypes.byref(n)) == 0
    assert n.value == 4096 * 2 * 16384 * 4
    assert lib.cs_workspace_bytes(1, 1 << 24, 1 << 22, 65536, 1, 0, None, ctypes.byref(n)) == 0
    assert n.value >= 4 * (1 << 24) * 4
    assert cs.REPORT_DTYPE.itemsize == 40


def test_create_ex_rejects_bad_psi(lib):
    """cs_operator_create_ex argument checks that run before any device work."""
    h = ctypes.c_void_p()
    assert lib.cs_operator_create_ex(1024, 256, 1, None, None, None, 7, None, 0, None, ctypes.byref(h)) == 1
    assert lib.cs_operator_create_ex(1024, 256, 1, None, None, None, 1, None, 0, None, ctypes.byref(h)) == 1


def test_missing_library_fails_loudly():
    """The product path has no fallback: without libcsgpu.so the binding raises."""
    import subprocess
    import sys
    code = ("import paper_1509_03979_b200 as cs\n"
            "try:\n"
            "    cs.load_library('/nonexistent/libcsgpu.so')\n"
            "except ImportError as e:\n"
            "    print('raised', e)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("raised"), r.stdout


def test_product_package_never_imports_the_oracle():
    """oracle/ is test infrastructure: the package (binding, dist helpers) must not reach it."""
    pkg = os.path.join(ROOT, "paper_1509_03979_b200")
    for f in sorted(os.listdir(pkg)):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f


def test_refine_workspace_sizes(lib):
    """refine_fp64 grows the recovery workspace by the refinement's share on the CTA tier, for
    the device-path and the host-buffer sizes alike; fp64 and Tier L sizes ignore it."""
    import paper_1509_03979_b200 as cs
    n0, n1, h0, h1 = (ctypes.c_size_t() for _ in range(4))
    o = cs.cs_options()
    o.refine_fp64 = 1
    B, N, M, K = 4096, 16384, 4096, 256
    assert lib.cs_workspace_bytes(1, N, M, K, B, 0, None, ctypes.byref(n0)) == 0
    assert lib.cs_workspace_bytes(1, N, M, K, B, 0, ctypes.byref(o), ctypes.byref(n1)) == 0
    cap = min(B, 256)
    # count + list + fp64 y + fp64 c0 (2N) + fp64 values + supports + reports, each 256-aligned
    assert n1.value >= n0.value + cap * (M * 8 + 2 * N * 8 + K * 12 + 40)
    assert lib.cs_workspace_bytes_host(1, N, M, K, B, 0, None, ctypes.byref(h0)) == 0
    assert lib.cs_workspace_bytes_host(1, N, M, K, B, 0, ctypes.byref(o), ctypes.byref(h1)) == 0
    assert h1.value - h0.value == n1.value - n0.value
    assert lib.cs_workspace_bytes(1, N, M, K, B, 1, ctypes.byref(o), ctypes.byref(n1)) == 0
    assert lib.cs_workspace_bytes(1, N, M, K, B, 1, None, ctypes.byref(n0)) == 0
    assert n1.value == n0.value
