"""paper_1509_03979_b200 — B200-native greedy compressive sensing (arXiv:1509.03979).

Thin ctypes binding over the C ABI of libcsgpu.so (include/cs.h).  It only
marshals arguments: every step of the method (operator, detection, CG-based
weighted least squares, pursuits) runs in the library's sm_100a kernels.
PyTorch supplies device memory and the current CUDA stream.

There is NO CPU fallback: if the shared library is missing or the device is
not a B200 the calls raise.

Names follow include/cs.h:
    cs_operator_create / cs_operator_apply / cs_operator_adjoint
    cs_recover / cs_recover_batched / cs_workspace_bytes
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcsgpu.so")

ALGS = {"omp": 0, "sp": 1, "ompr": 2, "cosamp": 3}
TERM_NAMES = {0: "done", 1: "iter_cap", 2: "stagnation", 3: "support_fixed", 4: "resid_rose"}
STATUS = {0: "CS_OK", 1: "CS_ERR_INVALID_ARG", 2: "CS_ERR_UNSUPPORTED", 3: "CS_ERR_WORKSPACE",
          4: "CS_ERR_CUDA", 5: "CS_ERR_NONFINITE"}

REPORT_DTYPE = np.dtype([("outer_iters", "<i4"), ("cg_iters_total", "<i4"), ("cg_solves", "<i4"),
                         ("applies", "<i4"), ("termination", "<i4"), ("status", "<u4"),
                         ("resid_norm", "<f8"), ("cg_rel_resid", "<f8")])
assert REPORT_DTYPE.itemsize == 40


class CsError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class cs_options(ctypes.Structure):
    _fields_ = [("max_outer", ctypes.c_int32), ("cg_max_iters", ctypes.c_int32),
                ("ompr_l", ctypes.c_int32), ("ompr_eta", ctypes.c_float),
                ("refine_fp64", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


_lib = None

EXPORTS = [
    "cs_operator_meta_bytes", "cs_operator_create", "cs_operator_destroy", "cs_operator_info",
    "cs_operator_ws_bytes", "cs_operator_apply", "cs_operator_apply_f64", "cs_operator_adjoint",
    "cs_operator_adjoint_f64", "cs_workspace_bytes", "cs_recover", "cs_recover_f64",
    "cs_recover_batched", "cs_recover_batched_f64", "cs_workspace_bytes_host", "cs_recover_batched_host",
    "cs_recover_batched_host_f64", "cs_status_string", "cs_last_error",
    "cs_launch_count", "cs_version", "cs_diag_phase_offset", "cs_diag_grid_barrier_us",
    "cs_dist_geometry", "cs_dist_ws_bytes", "cs_dist_phase", "cs_dist_copy", "cs_dist_row_offsets",
    "cs_diag_topk", "cs_diag_topk_grid", "cs_diag_topk_grid_ws_bytes", "cs_operator_meta_bytes_perm", "cs_operator_create_perm", "cs_operator_create_ex",
    "cs_operator_meta_bytes_ex", "cs_operator_meta_bytes_dft", "cs_operator_create_dft",
    "cs_support_to_dense", "cs_support_to_dense_f64", "cs_comm_init", "cs_gather_batched", "cs_gather_batched_after", "cs_comm_destroy",
]


def load_library(path: str = LIB_PATH):
    """Load libcsgpu.so and declare the signatures.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    sig = {
        "cs_operator_meta_bytes": (SZ, [I64, I64, I64]),
        "cs_operator_create": (I32, [I64, I64, I64, P, P, P, SZ, P, ctypes.POINTER(P)]),
        "cs_operator_meta_bytes_perm": (SZ, [I64, I64, I64]),
        "cs_operator_create_perm": (I32, [I64, I64, I64, P, P, P, P, SZ, P, ctypes.POINTER(P)]),
        "cs_operator_meta_bytes_ex": (SZ, [I64, I64, I64, ctypes.c_int, ctypes.c_int]),
        "cs_operator_meta_bytes_dft": (SZ, [I64, I64, I64]),
        "cs_support_to_dense": (I32, [I64, I64, I32, P, P, P, P]),
        "cs_support_to_dense_f64": (I32, [I64, I64, I32, P, P, P, P]),
        "cs_comm_init": (I32, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(P)]),
        "cs_gather_batched": (I32, [P, ctypes.c_int, I64, I32, ctypes.POINTER(P), ctypes.POINTER(P),
                                    ctypes.POINTER(P), P, P, P]),
        "cs_gather_batched_after": (I32, [P, ctypes.c_int, I64, I32, ctypes.POINTER(P), ctypes.POINTER(P),
                                          ctypes.POINTER(P), P, P, P, ctypes.POINTER(P)]),
        "cs_comm_destroy": (I32, [P]),
        "cs_operator_create_dft": (I32, [I64, I64, I64, P, P, P, P, SZ, P, ctypes.POINTER(P)]),
        "cs_operator_create_ex": (I32, [I64, I64, I64, P, P, P, ctypes.c_int, P, SZ, P, ctypes.POINTER(P)]),
        "cs_operator_destroy": (I32, [P]),
        "cs_operator_info": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "cs_operator_ws_bytes": (SZ, [P, ctypes.c_int]),
        "cs_operator_apply": (I32, [P, P, P, P, SZ, P]),
        "cs_operator_apply_f64": (I32, [P, P, P, P, SZ, P]),
        "cs_operator_adjoint": (I32, [P, P, P, P, SZ, P]),
        "cs_operator_adjoint_f64": (I32, [P, P, P, P, SZ, P]),
        "cs_workspace_bytes": (I32, [ctypes.c_int, I64, I64, I32, I64, ctypes.c_int,
                                     ctypes.POINTER(cs_options), ctypes.POINTER(SZ)]),
        "cs_recover": (I32, [P, ctypes.c_int, P, I64, I64, I32, ctypes.c_double,
                             ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_recover_f64": (I32, [P, ctypes.c_int, P, I64, I64, I32, ctypes.c_double,
                                 ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_recover_batched": (I32, [P, ctypes.c_int, P, I64, I64, I64, I32, ctypes.c_double,
                                     ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_recover_batched_f64": (I32, [P, ctypes.c_int, P, I64, I64, I64, I32, ctypes.c_double,
                                         ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_workspace_bytes_host": (I32, [ctypes.c_int, I64, I64, I32, I64, ctypes.c_int,
                                          ctypes.POINTER(cs_options), ctypes.POINTER(SZ)]),
        "cs_recover_batched_host": (I32, [P, ctypes.c_int, P, I64, I64, I64, I32, ctypes.c_double,
                                          ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_recover_batched_host_f64": (I32, [P, ctypes.c_int, P, I64, I64, I64, I32, ctypes.c_double,
                                              ctypes.POINTER(cs_options), P, P, P, P, SZ, P]),
        "cs_status_string": (ctypes.c_char_p, [I32]),
        "cs_last_error": (ctypes.c_char_p, []),
        "cs_launch_count": (ctypes.c_uint64, [ctypes.c_int]),
        "cs_version": (ctypes.c_char_p, []),
        "cs_diag_phase_offset": (I64, [ctypes.c_int, I64, I64, I32, I32, ctypes.c_int]),
        "cs_diag_grid_barrier_us": (ctypes.c_double, [ctypes.c_int, ctypes.c_int]),
        "cs_diag_topk": (I32, [P, I64, I64, ctypes.c_int, ctypes.c_int, P, P]),
        "cs_diag_topk_grid": (I32, [P, I64, I64, ctypes.c_int, P, P, SZ, P]),
        "cs_dist_geometry": (I32, [I64, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I32)]),
        "cs_dist_ws_bytes": (SZ, [I64, I64]),
        "cs_dist_phase": (I32, [P, ctypes.c_int, I64, I64, I64, I64, P, P, P, SZ, P]),
        "cs_dist_copy": (I32, [P, P, P, P, I64, I64, P, ctypes.c_int, P]),
        "cs_dist_row_offsets": (I32, [P, ctypes.POINTER(I64)]),
        "cs_diag_topk_grid_ws_bytes": (SZ, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        raise CsError(status, where, _lib.cs_last_error().decode())


def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def make_options(max_outer=0, cg_max_iters=0, ompr_l=0, ompr_eta=0.0) -> cs_options:
    o = cs_options()
    o.max_outer, o.cg_max_iters, o.ompr_l, o.ompr_eta = max_outer, cg_max_iters, ompr_l, ompr_eta
    return o


def launch_count(reset: bool = False) -> int:
    return int(load_library().cs_launch_count(1 if reset else 0))


class Operator:
    """Handle for A = P . DCT-II . diag(sigma) with `batch` independent instances; with
    `perm` ([batch][N] int32 pi), the Eq.(7) operator P . DCT-II . R . diag(sigma)
    (cs_operator_create_perm; sign_bits may then be None for sigma = +1)."""

    def __init__(self, N: int, M: int, sign_bits, rows, batch: int = 1, stream=None, perm=None, psi=None,
                 transform="dct"):
        torch = _torch()
        L = load_library()
        self.N, self.M, self.batch = int(N), int(M), int(batch)
        self.psi = psi
        dev = rows.device
        rw = rows.to(device=dev, dtype=torch.int32).contiguous()
        sb = None if sign_bits is None else sign_bits.to(device=dev).contiguous()
        h = ctypes.c_void_p()
        if transform == "dft":
            # partial Fourier (R36): `rows` are frequencies, M = 2 x their count
            nf = int(rw.shape[-1])
            if M != 2 * nf:
                raise ValueError("partial Fourier: M must be twice the number of frequencies")
            pm = None if perm is None else perm.to(device=dev, dtype=torch.int32).contiguous()
            nb = L.cs_operator_meta_bytes_dft(N, nf, batch)
            self.meta = torch.empty(nb, dtype=torch.uint8, device=dev)
            _check(L.cs_operator_create_dft(N, nf, batch, _ptr(sb) if sb is not None else None,
                                            _ptr(pm) if pm is not None else None, _ptr(rw), _ptr(self.meta),
                                            nb, _stream(stream), ctypes.byref(h)), "cs_operator_create_dft")
        elif psi is not None:
            code = {"I": 0, "dct": 1}[psi]
            pm = None if perm is None else perm.to(device=dev, dtype=torch.int32).contiguous()
            nb = L.cs_operator_meta_bytes_ex(N, M, batch, int(pm is not None), code)
            self.meta = torch.empty(nb, dtype=torch.uint8, device=dev)
            _check(L.cs_operator_create_ex(N, M, batch, _ptr(sb) if sb is not None else None,
                                           _ptr(pm) if pm is not None else None, _ptr(rw), code,
                                           _ptr(self.meta), nb, _stream(stream), ctypes.byref(h)),
                   "cs_operator_create_ex")
        elif perm is None:
            nb = L.cs_operator_meta_bytes(N, M, batch)
            self.meta = torch.empty(nb, dtype=torch.uint8, device=dev)
            _check(L.cs_operator_create(N, M, batch, _ptr(sb), _ptr(rw), _ptr(self.meta), nb,
                                        _stream(stream), ctypes.byref(h)), "cs_operator_create")
        else:
            pm = perm.to(device=dev, dtype=torch.int32).contiguous()
            nb = L.cs_operator_meta_bytes_perm(N, M, batch)
            self.meta = torch.empty(nb, dtype=torch.uint8, device=dev)
            _check(L.cs_operator_create_perm(N, M, batch, _ptr(sb) if sb is not None else None, _ptr(pm),
                                             _ptr(rw), _ptr(self.meta), nb, _stream(stream),
                                             ctypes.byref(h)), "cs_operator_create_perm")
        self.handle = h
        self._ws = {}

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.cs_operator_destroy(self.handle)
        except Exception:
            pass

    def ws(self, dtype):
        torch = _torch()
        prec = 1 if dtype == torch.float64 else 0
        nb = int(_lib.cs_operator_ws_bytes(self.handle, prec))
        if nb == 0:
            return None, 0
        key = (prec, nb)
        if key not in self._ws:
            self._ws[key] = torch.empty(nb, dtype=torch.uint8, device=self.meta.device)
        return self._ws[key], nb


def cs_operator_create(N, M, batch, sign_bits, rows, stream=None) -> Operator:
    return Operator(N, M, sign_bits, rows, batch, stream)


def cs_operator_apply(op: Operator, x, out=None, stream=None):
    """y[b] = A_b x[b]; x is [batch, N] (or [N]) float32/float64 on the GPU."""
    torch = _torch()
    x = x.contiguous()
    y = out if out is not None else torch.empty(x.shape[:-1] + (op.M,), dtype=x.dtype, device=x.device)
    ws, nb = op.ws(x.dtype)
    f = _lib.cs_operator_apply_f64 if x.dtype == torch.float64 else _lib.cs_operator_apply
    _check(f(op.handle, _ptr(x), _ptr(y), _ptr(ws) if ws is not None else None, nb, _stream(stream)),
           "cs_operator_apply")
    return y


def cs_operator_adjoint(op: Operator, y, out=None, stream=None):
    torch = _torch()
    y = y.contiguous()
    x = out if out is not None else torch.empty(y.shape[:-1] + (op.N,), dtype=y.dtype, device=y.device)
    ws, nb = op.ws(y.dtype)
    f = _lib.cs_operator_adjoint_f64 if y.dtype == torch.float64 else _lib.cs_operator_adjoint
    _check(f(op.handle, _ptr(y), _ptr(x), _ptr(ws) if ws is not None else None, nb, _stream(stream)),
           "cs_operator_adjoint")
    return x


def cs_workspace_bytes(alg, N, M, K, batch=1, dtype=None, opts: Optional[cs_options] = None) -> int:
    torch = _torch()
    L = load_library()
    n = ctypes.c_size_t()
    prec = 1 if dtype == torch.float64 else 0
    _check(L.cs_workspace_bytes(ALGS[alg] if isinstance(alg, str) else alg, N, M, K, batch, prec,
                                ctypes.byref(opts) if opts is not None else None, ctypes.byref(n)),
           "cs_workspace_bytes")
    return n.value


@dataclass
class Recovery:
    support: "object"   # torch int32 [.., K]
    values: "object"    # torch float [.., K]
    report_dev: "object"  # torch uint8 [.., 40] (device)

    def reports(self):
        raw = self.report_dev.cpu().numpy().reshape(-1, 40)
        return np.frombuffer(raw.tobytes(), dtype=REPORT_DTYPE)


class Workspace:
    """Caller-owned workspace reused across calls (torch is the allocator)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes, device):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


def cs_recover_batched(op: Operator, alg, Y, K: int, tol: float, opts: Optional[cs_options] = None,
                       workspace: Optional[Workspace] = None, out: Optional[Recovery] = None,
                       stream=None) -> Recovery:
    """Recover B = Y.shape[0] independent problems; problem b uses operator instance b."""
    torch = _torch()
    Y = Y.contiguous()
    B, M = Y.shape
    a = ALGS[alg] if isinstance(alg, str) else alg
    nb = cs_workspace_bytes(a, op.N, M, K, B, Y.dtype, opts)
    ws = (workspace or Workspace()).get(nb, Y.device)
    if out is None:
        out = Recovery(torch.empty((B, K), dtype=torch.int32, device=Y.device),
                       torch.empty((B, K), dtype=Y.dtype, device=Y.device),
                       torch.empty((B, 40), dtype=torch.uint8, device=Y.device))
    f = _lib.cs_recover_batched_f64 if Y.dtype == torch.float64 else _lib.cs_recover_batched
    _check(f(op.handle, a, _ptr(Y), B, M, op.N, K, tol,
             ctypes.byref(opts) if opts is not None else None, _ptr(out.values), _ptr(out.support),
             _ptr(out.report_dev), _ptr(ws), ws.numel(), _stream(stream)), "cs_recover_batched")
    return out


@dataclass
class HostRecovery:
    support: "object"   # torch int32 [B, K] (pinned host)
    values: "object"    # torch float [B, K] (pinned host)
    report_host: "object"  # torch uint8 [B, 40] (pinned host)

    def reports(self):
        return np.frombuffer(self.report_host.numpy().tobytes(), dtype=REPORT_DTYPE)


def cs_recover_batched_host(op: Operator, alg, Y_host, K: int, tol: float, opts: Optional[cs_options] = None,
                            workspace: Optional[Workspace] = None, out: Optional[HostRecovery] = None,
                            stream=None) -> HostRecovery:
    """End-to-end entry point: Y_host [B, M] in (pinned) host memory, results to pinned host
    memory; the copies overlap the recovery inside the library (cs_recover_batched_host)."""
    torch = _torch()
    B, M = Y_host.shape
    a = ALGS[alg] if isinstance(alg, str) else alg
    prec = 1 if Y_host.dtype == torch.float64 else 0
    n = ctypes.c_size_t()
    _check(load_library().cs_workspace_bytes_host(a, op.N, M, K, B, prec,
                                                  ctypes.byref(opts) if opts is not None else None,
                                                  ctypes.byref(n)), "cs_workspace_bytes_host")
    ws = (workspace or Workspace()).get(n.value, op.meta.device)
    if out is None:
        out = HostRecovery(torch.empty((B, K), dtype=torch.int32).pin_memory(),
                           torch.empty((B, K), dtype=Y_host.dtype).pin_memory(),
                           torch.empty((B, 40), dtype=torch.uint8).pin_memory())
    f = _lib.cs_recover_batched_host_f64 if prec else _lib.cs_recover_batched_host
    _check(f(op.handle, a, _ptr(Y_host), B, M, op.N, K, tol,
             ctypes.byref(opts) if opts is not None else None, _ptr(out.values), _ptr(out.support),
             _ptr(out.report_host), _ptr(ws), ws.numel(), _stream(stream)), "cs_recover_batched_host")
    return out


def cs_recover(op: Operator, alg, y, M: int, N: int, K: int, tol: float,
               opts: Optional[cs_options] = None, workspace: Optional[Workspace] = None,
               stream=None) -> Recovery:
    """Single-signal recovery (operator instance 0)."""
    torch = _torch()
    y = y.contiguous()
    a = ALGS[alg] if isinstance(alg, str) else alg
    nb = cs_workspace_bytes(a, N, M, K, 1, y.dtype, opts)
    ws = (workspace or Workspace()).get(nb, y.device)
    out = Recovery(torch.empty(K, dtype=torch.int32, device=y.device),
                   torch.empty(K, dtype=y.dtype, device=y.device),
                   torch.empty(40, dtype=torch.uint8, device=y.device))
    f = _lib.cs_recover_f64 if y.dtype == torch.float64 else _lib.cs_recover
    _check(f(op.handle, a, _ptr(y), M, N, K, tol, ctypes.byref(opts) if opts is not None else None,
             _ptr(out.values), _ptr(out.support), _ptr(out.report_dev), _ptr(ws), ws.numel(),
             _stream(stream)), "cs_recover")
    return out


def cs_support_to_dense(support, values, N: int, stream=None):
    """Dense [B][N] signals from (support, values) of a recovery (cs_support_to_dense)."""
    torch = _torch()
    B, K = support.shape
    out = torch.empty((B, N), dtype=values.dtype, device=values.device)
    f = _lib.cs_support_to_dense_f64 if values.dtype == torch.float64 else _lib.cs_support_to_dense
    _check(f(B, N, K, _ptr(support.contiguous()), _ptr(values.contiguous()), _ptr(out), _stream(stream)),
           "cs_support_to_dense")
    return out


class Comm:
    """Single-process multi-GPU results gather (cs_comm_init / cs_gather_batched)."""

    def __init__(self, devices):
        load_library()
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        _check(_lib.cs_comm_init(len(self.devices), arr, ctypes.byref(h)), "cs_comm_init")
        self.handle = h

    def gather(self, results, root: int = 0):
        """results: one Recovery per device (same B, K; fp32), in `devices` order.  Returns the
        root's concatenated (support, values, raw reports) tensors."""
        torch = _torch()
        nd = len(self.devices)
        B, K = results[0].support.shape
        dev = results[root].support.device
        vals = torch.empty((nd * B, K), dtype=torch.float32, device=dev)
        supp = torch.empty((nd * B, K), dtype=torch.int32, device=dev)
        reps = torch.empty((nd * B, 40), dtype=torch.uint8, device=dev)
        P = ctypes.c_void_p
        pv = (P * nd)(*[r.values.data_ptr() for r in results])
        ps = (P * nd)(*[r.support.data_ptr() for r in results])
        pr = (P * nd)(*[r.report_dev.data_ptr() for r in results])
        # ordered after each device's current torch stream (the producers of the records and
        # of the freshly allocated outputs): no host synchronisation needed before the call
        after = (P * nd)(*[torch.cuda.current_stream(d).cuda_stream for d in self.devices])
        _check(_lib.cs_gather_batched_after(self.handle, root, B, K, pv, ps, pr, _ptr(vals), _ptr(supp),
                                            _ptr(reps), after), "cs_gather_batched_after")
        return supp, vals, reps

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.cs_comm_destroy(self.handle)
        except Exception:
            pass
