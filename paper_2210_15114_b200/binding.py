"""Thin Python binding of the C ABI in include/l1dm.h (ctypes; argument marshalling only).

Every step of the hot path runs in libl1dm.so's sm_100a kernels.  There is no CPU
fallback: if the library is missing the import of this module's functions raises,
and on a machine without an sm_100 device the library itself returns L1DM_EDEVICE.

Names mirror the C entry points: l1dm_prepare / l1dm_matvec / l1dm_free (BASELINE.json
north_star), plus the _ex shard/stream variants and the introspection calls.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("L1DM_LIB") or os.path.join(_PKG, "lib", "libl1dm.so")

STATUS = {
    0: "L1DM_OK", -1: "L1DM_EINVAL", -2: "L1DM_ENONFINITE", -3: "L1DM_ENOMEM",
    -4: "L1DM_ECUDA", -5: "L1DM_EDEVICE", -6: "L1DM_ENOTIMPL", -7: "L1DM_ETIMEOUT",
    -8: "L1DM_ENOTSIMPLEX",
}

EXPORTS = [
    "l1dm_prepare", "l1dm_prepare_ex", "l1dm_matvec", "l1dm_matvec_ex", "l1dm_matvec_pipelined",
    "l1dm_matvec_lp", "l1dm_matvec_lp_ex", "l1dm_tv_matvec", "l1dm_tv_matvec_ex",
    "l1dm_lpp_even_matvec", "l1dm_bilinear_matvec", "l1dm_l2_embed", "l1dm_query_layout",
    "l1dm_query_strategy",
    "l1dm_matvec_colblocks", "l1dm_unblock",
    "l1dm_free", "l1dm_sync",
    "l1dm_shape", "l1dm_workspace_bytes", "l1dm_set_workspace_limit", "l1dm_set_query_mode",
    "l1dm_plan", "l1dm_plan_ex", "l1dm_timing_enable", "l1dm_timing_read", "l1dm_debug_export", "l1dm_release_cached",
    "l1dm_ipc_alloc", "l1dm_ipc_free", "l1dm_ipc_open", "l1dm_ipc_close", "l1dm_matvec_push",
    "l1dm_peer_reduce", "l1dm_peer_wait", "l1dm_peer_check",
    "l1dm_last_error", "l1dm_handleless_launches", "l1dm_version",
    "l1dm_gemm", "l1dm_syevj", "l1dm_syev_topk", "l1dm_op_apply", "l1dm_block_krylov", "l1dm_cg",
    "l1dm_block_krylov_cb", "l1dm_cg_cb",
]


class L1dmError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class PlanT(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in (
        "mb", "col_blocks", "vec", "lanes_per_row", "rows_per_tile", "tiles_per_segment", "kc",
        "chunks", "l2_resident", "workspace_bytes", "scatter")]


MAX_PEERS = 16


class PeerT(ctypes.Structure):
    """l1dm_peer_t (include/l1dm.h): the peer buffers of one rank's group, as mapped here."""
    _fields_ = [("world", ctypes.c_int), ("rank", ctypes.c_int),
                ("inbox", ctypes.c_void_p * MAX_PEERS), ("flags", ctypes.c_void_p * MAX_PEERS),
                ("ybuf", ctypes.c_void_p * MAX_PEERS), ("timeout", ctypes.c_void_p),
                ("n", ctypes.c_int64), ("m", ctypes.c_int64)]


class OperatorT(ctypes.Structure):
    """l1dm_operator_t (include/l1dm.h): the matrix the NEXT-2 consumers apply."""
    _fields_ = [("kind", ctypes.c_int), ("p", ctypes.c_int), ("h", ctypes.c_void_p),
                ("X", ctypes.c_void_p), ("n", ctypes.c_int64), ("ld_x", ctypes.c_int64),
                ("d", ctypes.c_int64), ("M", ctypes.c_void_p)]


class KrylovInfoT(ctypes.Structure):
    _fields_ = [("products", ctypes.c_int64), ("columns", ctypes.c_int64),
                ("block", ctypes.c_int64), ("depth", ctypes.c_int64),
                ("product_ms", ctypes.c_double), ("total_ms", ctypes.c_double)]


class CGInfoT(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("residual", ctypes.c_double),
                ("converged", ctypes.c_int), ("products", ctypes.c_int64)]


APPLY_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class TimingT(ctypes.Structure):
    _fields_ = [("prep_ms", ctypes.c_double), ("colsums_ms", ctypes.c_double),
                ("scan_ms", ctypes.c_double), ("accumulate_ms", ctypes.c_double),
                ("copy_ms", ctypes.c_double), ("colsums_launches", ctypes.c_int64),
                ("scan_launches", ctypes.c_int64), ("accumulate_launches", ctypes.c_int64),
                ("queries", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("scan_pairs", ctypes.c_int64), ("accumulate_pairs", ctypes.c_int64),
                ("m_last", ctypes.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libl1dm.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libl1dm.so not found at {path}; run "
                          "`python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    st = ctypes.c_int
    lib.l1dm_prepare.argtypes = [vp, i64, i64, ctypes.POINTER(vp)]
    lib.l1dm_prepare_ex.argtypes = [vp, i64, i64, i64, i64, vp, ctypes.POINTER(vp)]
    lib.l1dm_matvec.argtypes = [vp, vp, i64, vp]
    lib.l1dm_matvec_ex.argtypes = [vp, vp, i64, i64, vp, i64, vp]
    lib.l1dm_matvec_lp_ex.argtypes = [vp, i32, vp, i64, i64, vp, i64, vp]
    lib.l1dm_matvec_lp.argtypes = [vp, i32, vp, i64, vp]
    lib.l1dm_tv_matvec_ex.argtypes = [vp, vp, i64, i64, vp, i64, vp]
    lib.l1dm_tv_matvec.argtypes = [vp, vp, i64, vp]
    lib.l1dm_lpp_even_matvec.argtypes = [vp, i64, i64, i64, i32, vp, i64, i64, vp, i64, vp]
    lib.l1dm_bilinear_matvec.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, vp, i64, vp]
    lib.l1dm_l2_embed.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, vp]
    lib.l1dm_query_strategy.argtypes = [vp, i64, ctypes.POINTER(i32)]
    lib.l1dm_query_strategy.restype = st
    lib.l1dm_query_layout.argtypes = [vp, i64, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                      ctypes.POINTER(i64)]
    lib.l1dm_matvec_colblocks.argtypes = [vp, vp, i64, i64, vp, vp, i64, ctypes.POINTER(vp)]
    lib.l1dm_unblock.argtypes = [vp, i64, i64, i64, vp, i64, vp]
    lib.l1dm_matvec_pipelined.argtypes = [vp, vp, i64, i64, vp, i64, vp, i64,
                                           ctypes.POINTER(vp)]
    lib.l1dm_free.argtypes = [vp]
    lib.l1dm_free.restype = None
    lib.l1dm_sync.argtypes = [vp]
    lib.l1dm_shape.argtypes = [vp] + [ctypes.POINTER(i64)] * 4
    lib.l1dm_workspace_bytes.argtypes = [vp, i64]
    lib.l1dm_workspace_bytes.restype = ctypes.c_size_t
    lib.l1dm_set_workspace_limit.argtypes = [vp, ctypes.c_size_t]
    lib.l1dm_set_query_mode.argtypes = [vp, i32]
    lib.l1dm_plan.argtypes = [i64, i64, i64, i64, i64, ctypes.POINTER(PlanT)]
    lib.l1dm_plan_ex.argtypes = [i64, i64, i64, i64, i64, i32, ctypes.POINTER(PlanT)]
    lib.l1dm_timing_enable.argtypes = [vp, i32]
    lib.l1dm_timing_read.argtypes = [vp, ctypes.POINTER(TimingT), i32]
    lib.l1dm_debug_export.argtypes = [vp, vp, vp, vp, vp]
    lib.l1dm_release_cached.argtypes = []
    lib.l1dm_release_cached.restype = st
    lib.l1dm_last_error.argtypes = []
    lib.l1dm_last_error.restype = ctypes.c_char_p
    lib.l1dm_ipc_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(vp), ctypes.c_char_p]
    lib.l1dm_ipc_free.argtypes = [vp]
    lib.l1dm_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.l1dm_ipc_close.argtypes = [vp]
    lib.l1dm_matvec_push.argtypes = [vp, vp, i64, i64, ctypes.POINTER(PeerT), ctypes.c_uint, vp]
    lib.l1dm_peer_reduce.argtypes = [ctypes.POINTER(PeerT), i64, i64, ctypes.c_uint, ctypes.c_uint,
                                     vp]
    lib.l1dm_peer_wait.argtypes = [ctypes.POINTER(PeerT), ctypes.c_uint, i64, i64, vp, i64, vp]
    lib.l1dm_peer_check.argtypes = [ctypes.POINTER(PeerT), vp]
    for name in ("l1dm_ipc_alloc", "l1dm_ipc_free", "l1dm_ipc_open", "l1dm_ipc_close",
                 "l1dm_matvec_push", "l1dm_peer_reduce", "l1dm_peer_wait", "l1dm_peer_check"):
        getattr(lib, name).restype = st
    dbl = ctypes.c_double
    lib.l1dm_gemm.argtypes = [i32, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp]
    lib.l1dm_syevj.argtypes = [i64, vp, i64, vp, vp, i64, vp]
    lib.l1dm_syev_topk.argtypes = [i64, vp, i64, i64, vp, vp, i64, vp]
    lib.l1dm_op_apply.argtypes = [ctypes.POINTER(OperatorT), vp, i64, i64, vp, i64, vp]
    lib.l1dm_block_krylov.argtypes = [ctypes.POINTER(OperatorT), i64, i64, i64, vp, vp, vp, vp,
                                      i64, vp, ctypes.POINTER(KrylovInfoT)]
    lib.l1dm_cg.argtypes = [ctypes.POINTER(OperatorT), vp, vp, dbl, i64, i32, vp,
                            ctypes.POINTER(CGInfoT)]
    lib.l1dm_block_krylov_cb.argtypes = [i64, APPLY_FN, vp, i64, i64, i64, vp, vp, vp, vp, i64, vp,
                                         ctypes.POINTER(KrylovInfoT)]
    lib.l1dm_cg_cb.argtypes = [i64, APPLY_FN, vp, vp, vp, dbl, i64, i32, vp, ctypes.POINTER(CGInfoT)]
    for name in ("l1dm_gemm", "l1dm_syevj", "l1dm_syev_topk", "l1dm_op_apply", "l1dm_block_krylov",
                 "l1dm_cg", "l1dm_block_krylov_cb", "l1dm_cg_cb"):
        getattr(lib, name).restype = st
    lib.l1dm_handleless_launches.argtypes = []
    lib.l1dm_handleless_launches.restype = i64
    lib.l1dm_version.argtypes = []
    lib.l1dm_version.restype = ctypes.c_char_p
    for name in ("l1dm_prepare", "l1dm_prepare_ex", "l1dm_matvec", "l1dm_matvec_ex",
                 "l1dm_matvec_pipelined", "l1dm_sync", "l1dm_matvec_lp", "l1dm_matvec_lp_ex",
                 "l1dm_tv_matvec", "l1dm_tv_matvec_ex", "l1dm_lpp_even_matvec",
                 "l1dm_bilinear_matvec", "l1dm_l2_embed", "l1dm_query_layout",
                 "l1dm_matvec_colblocks", "l1dm_unblock",
                 "l1dm_shape", "l1dm_set_workspace_limit", "l1dm_set_query_mode", "l1dm_plan", "l1dm_plan_ex",
                 "l1dm_timing_enable",
                 "l1dm_timing_read", "l1dm_debug_export"):
        getattr(lib, name).restype = st
    _lib = lib
    return lib


def _check(rc: int, where: str):
    if rc != 0:
        raise L1dmError(rc, where, load_library().l1dm_last_error().decode())


def _ptr(t) -> ctypes.c_void_p:
    if isinstance(t, torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)


def _stream_of(t, stream):
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    if isinstance(t, torch.Tensor) and t.is_cuda:
        return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    return ctypes.c_void_p(0)


def _as_f32_2d(A, name):
    if isinstance(A, np.ndarray):
        A = torch.from_numpy(np.ascontiguousarray(A))
    if A.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {A.dtype}")
    if A.dim() == 1:
        A = A.view(-1, 1)
    if A.dim() != 2 or A.stride(1) != 1:
        A = A.contiguous()
    return A


@dataclass
class Handle:
    """An l1dm_handle: prepared state for coordinates [k_begin, k_end) of n points."""
    ptr: ctypes.c_void_p
    n: int
    d_local: int
    k_begin: int
    k_end: int
    device: int

    def __del__(self):
        if self.ptr:
            try:
                load_library().l1dm_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


def l1dm_prepare(X, k_begin: int = 0, k_end: int | None = None, stream=None) -> Handle:
    """Alg. 1: sort every coordinate of X (n x d fp32; host or CUDA tensor)."""
    lib = load_library()
    X = _as_f32_2d(X, "X")
    n, d = X.shape
    if k_end is None:
        k_end = d
    out = ctypes.c_void_p()
    if X.is_cuda:
        with torch.cuda.device(X.device):
            rc = lib.l1dm_prepare_ex(_ptr(X), n, X.stride(0), k_begin, k_end,
                                     _stream_of(X, stream), ctypes.byref(out))
        dev = X.device.index
    else:
        rc = lib.l1dm_prepare_ex(_ptr(X), n, X.stride(0), k_begin, k_end,
                                 _stream_of(X, stream), ctypes.byref(out))
        dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    _check(rc, "l1dm_prepare")
    return Handle(out, n, k_end - k_begin, k_begin, k_end, dev)


def _query(entry: str, extra: tuple, h: Handle, Z, Y, stream, block=True):
    lib = load_library()
    squeeze = (Z.ndim == 1)
    Z = _as_f32_2d(Z, "Z")
    if Z.shape[0] != h.n:
        raise ValueError(f"Z has {Z.shape[0]} rows, handle has n={h.n}")
    m = Z.shape[1]
    if Y is None:
        Y = torch.empty((h.n, m), dtype=torch.float64, device=Z.device)
    elif isinstance(Y, np.ndarray):
        Y = torch.from_numpy(Y)
    if Y.dtype != torch.float64 or Y.dim() != 2 or Y.shape != (h.n, m) or Y.stride(1) != 1:
        raise ValueError("Y must be an n x m float64 row-major tensor")
    fn = getattr(lib, entry)
    if Z.is_cuda:
        with torch.cuda.device(Z.device):
            rc = fn(h.ptr, *extra, _ptr(Z), Z.stride(0), m, _ptr(Y), Y.stride(0),
                    _stream_of(Z, stream))
    else:
        rc = fn(h.ptr, *extra, _ptr(Z), Z.stride(0), m, _ptr(Y), Y.stride(0), _stream_of(Z, stream))
        _check(rc, entry.replace("_ex", ""))
        if block:  # pinned host buffers run asynchronously in the library (include/l1dm.h)
            l1dm_sync(h)
    _check(rc, entry.replace("_ex", ""))
    return Y.view(-1) if squeeze else Y


def l1dm_matvec(h: Handle, Z, Y=None, stream=None, block=True):
    """Alg. 2 for the m columns of Z: returns Y = A·Z (fp64, n x m).

    CUDA tensors: stream-ordered on `stream` (default: torch's current stream).
    Host tensors / numpy arrays: staged through device buffers; synchronous unless Z and Y are
    pinned and block=False (then the copies of consecutive calls overlap the compute, and the
    caller runs l1dm_sync before reading Y)."""
    return _query("l1dm_matvec_ex", (), h, Z, Y, stream, block)


def l1dm_matvec_lp(h: Handle, p: int, Z, Y=None, stream=None, block=True):
    """l_p^p block product for odd p in {1, 3, 5, 7} (Thm. odd_p): sum_k |x_ik - x_jk|^p."""
    return _query("l1dm_matvec_lp_ex", (int(p),), h, Z, Y, stream, block)


def l1dm_tv_matvec(h: Handle, Z, Y=None, stream=None):
    """Total-variation block product (Thm. tv) for rows on the probability simplex."""
    return _query("l1dm_tv_matvec_ex", (), h, Z, Y, stream)


def l1dm_lpp_even_matvec(X, p: int, Z, Y=None, stream=None):
    """Sort-free even-p l_p^p block product (p in {2, 4, 6}; p = 2: squared Euclidean).
    No preprocessing: X (n x d) is read by the call."""
    lib = load_library()
    X = _as_f32_2d(X, "X")
    squeeze = (Z.ndim == 1)
    Z = _as_f32_2d(Z, "Z")
    n, d = X.shape
    if Z.shape[0] != n:
        raise ValueError(f"Z has {Z.shape[0]} rows, X has {n}")
    m = Z.shape[1]
    if Y is None:
        Y = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    if Y.dtype != torch.float64 or Y.shape != (n, m) or Y.stride(1) != 1:
        raise ValueError("Y must be an n x m float64 row-major tensor")
    dev = Z.device if Z.is_cuda else (X.device if X.is_cuda else None)
    if dev is not None:
        with torch.cuda.device(dev):
            rc = lib.l1dm_lpp_even_matvec(_ptr(X), n, X.stride(0), d, int(p), _ptr(Z), Z.stride(0),
                                          m, _ptr(Y), Y.stride(0), _stream_of(Z, stream))
    else:
        rc = lib.l1dm_lpp_even_matvec(_ptr(X), n, X.stride(0), d, int(p), _ptr(Z), Z.stride(0), m,
                                      _ptr(Y), Y.stride(0), _stream_of(Z, stream))
    _check(rc, "l1dm_lpp_even_matvec")
    return Y.view(-1) if squeeze else Y


def l1dm_bilinear_matvec(X, M, Z, Y=None, stream=None):
    """Thm. maha's bilinear form A_ij = x_i^T M x_j (M: d x d float64): Y = X M X^T Z."""
    lib = load_library()
    X = _as_f32_2d(X, "X")
    squeeze = (Z.ndim == 1)
    Z = _as_f32_2d(Z, "Z")
    M = torch.as_tensor(M)
    n, d = X.shape
    if M.dtype != torch.float64 or tuple(M.shape) != (d, d):
        raise ValueError("M must be a d x d float64 matrix")
    M = M.contiguous()
    if Z.shape[0] != n:
        raise ValueError(f"Z has {Z.shape[0]} rows, X has {n}")
    m = Z.shape[1]
    if Y is None:
        Y = torch.empty((n, m), dtype=torch.float64, device=Z.device)
    if Y.dtype != torch.float64 or Y.shape != (n, m) or Y.stride(1) != 1:
        raise ValueError("Y must be an n x m float64 row-major tensor")
    dev = Z.device if Z.is_cuda else (X.device if X.is_cuda else None)
    args = (_ptr(X), n, X.stride(0), d, _ptr(M), _ptr(Z), Z.stride(0), m, _ptr(Y), Y.stride(0),
            _stream_of(Z, stream))
    if dev is not None:
        with torch.cuda.device(dev):
            rc = lib.l1dm_bilinear_matvec(*args)
    else:
        rc = lib.l1dm_bilinear_matvec(*args)
    _check(rc, "l1dm_bilinear_matvec")
    return Y.view(-1) if squeeze else Y


def l1dm_l2_embed(X: torch.Tensor, G: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """Thm. l2embed: X' = X G^T / (beta k) (n x k fp32), X and G CUDA fp32 tensors."""
    lib = load_library()
    X = _as_f32_2d(X, "X")
    G = _as_f32_2d(G, "G").contiguous()
    n, d = X.shape
    k = G.shape[0]
    if G.shape[1] != d or not (X.is_cuda and G.is_cuda):
        raise ValueError("G must be k x d and X, G CUDA tensors")
    if out is None:
        out = torch.empty((n, k), dtype=torch.float32, device=X.device)
    with torch.cuda.device(X.device):
        rc = lib.l1dm_l2_embed(_ptr(X), n, X.stride(0), d, _ptr(G), k, _ptr(out), out.stride(0),
                               _stream_of(X, stream))
    _check(rc, "l1dm_l2_embed")
    return out


def l1dm_query_layout(h: Handle, m: int):
    """(scatter, mb, col_blocks) of the handle's plan for m columns."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(load_library().l1dm_query_layout(h.ptr, m, ctypes.byref(a), ctypes.byref(b),
                                            ctypes.byref(c)), "l1dm_query_layout")
    return a.value, b.value, c.value


def _event_handles(events, device, stream):
    out = []
    for e in events:
        if e.cuda_event == 0:  # torch creates the CUDA event lazily, on first record
            e.record(torch.cuda.current_stream(device) if stream is None else stream)
        out.append(ctypes.c_void_p(e.cuda_event))
    return (ctypes.c_void_p * len(out))(*out)


def l1dm_matvec_colblocks(h: Handle, Z: torch.Tensor, Yb: torch.Tensor, events, stream=None):
    """Scatter-strategy query into the column-block-major Yb (col_blocks x n x mb fp64, CUDA),
    recording events[cb] once block cb is final (include/l1dm.h)."""
    Z = _as_f32_2d(Z, "Z")
    if not (Z.is_cuda and Yb.is_cuda) or Yb.dtype != torch.float64 or not Yb.is_contiguous():
        raise ValueError("Z and Yb must be CUDA tensors; Yb contiguous float64")
    arr = _event_handles(events, Z.device, stream)
    with torch.cuda.device(Z.device):
        rc = load_library().l1dm_matvec_colblocks(h.ptr, _ptr(Z), Z.stride(0), Z.shape[1],
                                                  _ptr(Yb), _stream_of(Z, stream), len(events),
                                                  arr)
    _check(rc, "l1dm_matvec_colblocks")
    return Yb


def l1dm_unblock(Yb: torch.Tensor, m: int, Y: torch.Tensor, stream=None):
    """Row-major Y (n x m) from the column-block-major Yb (col_blocks x n x mb)."""
    n, mb = Yb.shape[1], Yb.shape[2]
    with torch.cuda.device(Yb.device):
        rc = load_library().l1dm_unblock(_ptr(Yb), n, m, mb, _ptr(Y), Y.stride(0),
                                         _stream_of(Yb, stream))
    _check(rc, "l1dm_unblock")
    return Y


def point_blocks(n: int, nblocks: int):
    """Row ranges [floor(b n / B), floor((b+1) n / B)) used by l1dm_matvec_pipelined."""
    return [((n * b) // nblocks, (n * (b + 1)) // nblocks) for b in range(nblocks)]


def l1dm_matvec_pipelined(h: Handle, Z: torch.Tensor, Y: torch.Tensor, events, stream=None):
    """As l1dm_matvec (CUDA tensors), recording events[b] once rows point_blocks(n, B)[b]
    of Y are final, so a collective on those rows can start while the rest is computed."""
    lib = load_library()
    Z = _as_f32_2d(Z, "Z")
    m = Z.shape[1]
    if not (Z.is_cuda and Y.is_cuda):
        raise ValueError("l1dm_matvec_pipelined needs CUDA tensors")
    if Y.dtype != torch.float64 or Y.shape != (h.n, m) or Y.stride(1) != 1:
        raise ValueError("Y must be an n x m float64 row-major tensor")
    st = _stream_of(Z, stream)
    handles = []
    for e in events:
        if e.cuda_event == 0:  # torch creates the CUDA event lazily, on first record
            e.record(torch.cuda.current_stream(Z.device) if stream is None else stream)
        handles.append(ctypes.c_void_p(e.cuda_event))
    arr = (ctypes.c_void_p * len(handles))(*handles)
    with torch.cuda.device(Z.device):
        rc = lib.l1dm_matvec_pipelined(h.ptr, _ptr(Z), Z.stride(0), m, _ptr(Y), Y.stride(0), st,
                                       len(handles), arr)
    _check(rc, "l1dm_matvec_pipelined")
    return Y


def l1dm_free(h: Handle):
    if h is not None and h.ptr:
        load_library().l1dm_free(h.ptr)
        h.ptr = None


def l1dm_sync(h: Handle):
    _check(load_library().l1dm_sync(h.ptr), "l1dm_sync")


def l1dm_set_workspace_limit(h: Handle, nbytes: int):
    _check(load_library().l1dm_set_workspace_limit(h.ptr, int(nbytes)), "l1dm_set_workspace_limit")


MODES = {"auto": 0, "gather": 1, "scatter": 2, "runs": 3}


def l1dm_set_query_mode(h: Handle, mode):
    """"auto" | "gather" | "scatter" (or 0/1/2): the query strategy, include/l1dm.h."""
    _check(load_library().l1dm_set_query_mode(h.ptr, MODES.get(mode, mode)), "l1dm_set_query_mode")


def l1dm_workspace_bytes(h: Handle, m: int) -> int:
    return int(load_library().l1dm_workspace_bytes(h.ptr, m))


def l1dm_plan(n: int, d_local: int, m: int, l2_bytes: int = 126 << 20, workspace_limit: int = 0,
              mode="auto"):
    """The query plan for these sizes (pure host function; mode "auto" | "gather" | "scatter")."""
    p = PlanT()
    _check(load_library().l1dm_plan_ex(n, d_local, m, l2_bytes, workspace_limit,
                                       MODES.get(mode, mode), ctypes.byref(p)), "l1dm_plan")
    return {f: getattr(p, f) for f, _ in PlanT._fields_}


def l1dm_timing_enable(h: Handle, enable: bool = True):
    _check(load_library().l1dm_timing_enable(h.ptr, 1 if enable else 0), "l1dm_timing_enable")


def l1dm_timing_read(h: Handle, reset: bool = False) -> dict:
    t = TimingT()
    _check(load_library().l1dm_timing_read(h.ptr, ctypes.byref(t), 1 if reset else 0),
           "l1dm_timing_read")
    return {f: getattr(t, f) for f, _ in TimingT._fields_}


def l1dm_debug_export(h: Handle):
    """Test-only: (sval, perm, rank) as d_local x n host arrays and hsum (n)."""
    sval = np.empty((h.d_local, h.n), dtype=np.float32)
    perm = np.empty((h.d_local, h.n), dtype=np.uint32)
    rank = np.empty((h.d_local, h.n), dtype=np.uint32)
    hs = np.empty(h.n, dtype=np.float64)
    _check(load_library().l1dm_debug_export(h.ptr, _ptr(sval), _ptr(perm), _ptr(rank), _ptr(hs)),
           "l1dm_debug_export")
    return sval, perm, rank, hs


def l1dm_release_cached():
    """Return cached device blocks of freed handles to CUDA (current device)."""
    _check(load_library().l1dm_release_cached(), "l1dm_release_cached")


# ------------------------------------------------------------ peer-memory collective (§8)
IPC_HANDLE_BYTES = 64


def l1dm_ipc_alloc(nbytes: int) -> tuple[int, bytes]:
    """Zeroed device allocation of nbytes on the current device and its CUDA IPC handle."""
    p = ctypes.c_void_p()
    hbuf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(load_library().l1dm_ipc_alloc(int(nbytes), ctypes.byref(p), hbuf), "l1dm_ipc_alloc")
    return int(p.value), bytes(hbuf.raw)


def l1dm_ipc_free(ptr: int):
    _check(load_library().l1dm_ipc_free(ctypes.c_void_p(ptr)), "l1dm_ipc_free")


def l1dm_ipc_open(handle: bytes) -> int:
    """Map another process's l1dm_ipc_alloc buffer (same node) into this one."""
    p = ctypes.c_void_p()
    _check(load_library().l1dm_ipc_open(handle, ctypes.byref(p)), "l1dm_ipc_open")
    return int(p.value)


def l1dm_ipc_close(ptr: int):
    _check(load_library().l1dm_ipc_close(ctypes.c_void_p(ptr)), "l1dm_ipc_close")


def l1dm_matvec_push(h: Handle, Z: torch.Tensor, peers: PeerT, epoch: int, stream=None):
    """This rank's partial A^(K_g) Z into the owners' inboxes, then its arrival flags."""
    Z = _as_f32_2d(Z, "Z")
    if not Z.is_cuda:
        raise ValueError("l1dm_matvec_push needs a CUDA Z")
    with torch.cuda.device(Z.device):
        rc = load_library().l1dm_matvec_push(h.ptr, _ptr(Z), Z.stride(0), Z.shape[1],
                                             ctypes.byref(peers), int(epoch),
                                             _stream_of(Z, stream))
    _check(rc, "l1dm_matvec_push")


def l1dm_peer_reduce(peers: PeerT, n: int, m: int, epoch: int, targets: int, stream=None):
    """Owner side: sum this rank's rows over the G slots into every target's result buffer."""
    _check(load_library().l1dm_peer_reduce(ctypes.byref(peers), n, m, int(epoch), int(targets),
                                           _stream_of(None, stream)), "l1dm_peer_reduce")


def l1dm_peer_wait(peers: PeerT, epoch: int, n: int, m: int, Y=None, stream=None):
    """Result side: wait for every owner's rows; copy the result into Y (CUDA, n x m fp64)."""
    yp, ldy = (ctypes.c_void_p(0), m) if Y is None else (_ptr(Y), Y.stride(0))
    if Y is not None and (Y.dtype != torch.float64 or not Y.is_cuda or tuple(Y.shape) != (n, m)):
        raise ValueError("Y must be a CUDA float64 n x m tensor")
    _check(load_library().l1dm_peer_wait(ctypes.byref(peers), int(epoch), n, m, yp, ldy,
                                         _stream_of(Y, stream)), "l1dm_peer_wait")


def l1dm_peer_check(peers: PeerT, stream=None):
    """Synchronise and raise L1dmError(ETIMEOUT) if a peer wait gave up."""
    _check(load_library().l1dm_peer_check(ctypes.byref(peers), _stream_of(None, stream)),
           "l1dm_peer_check")


STRATEGIES = {0: "gather", 1: "scatter", 2: "runs"}


def l1dm_query_strategy(h: Handle, m: int) -> str:
    """'gather', 'scatter' or 'runs': what an m-column l1 query on h runs."""
    v = ctypes.c_int()
    _check(load_library().l1dm_query_strategy(h.ptr, int(m), ctypes.byref(v)),
           "l1dm_query_strategy")
    return STRATEGIES[v.value]


def l1dm_handleless_launches() -> int:
    """Kernels launched so far by the handle-free entries (even p, bilinear, l2 embed)."""
    return int(load_library().l1dm_handleless_launches())


def l1dm_version() -> str:
    return load_library().l1dm_version().decode()


# ------------------------------------------------------------ matrix-free consumers (NEXT-2)
OP_SORTED, OP_EVEN, OP_BILINEAR = 0, 1, 2


class Operator:
    """The matrix A of a NEXT-2 consumer (include/l1dm.h l1dm_operator_t), touched only through
    the library's block product: a prepared handle (l1 or odd l_p^p), sort-free even l_p^p on
    device X, or the bilinear form x_i^T M x_j.  Keeps its tensors alive."""

    def __init__(self, kind: int, n: int, device, *, handle: Handle | None = None, p: int = 1,
                 X: torch.Tensor | None = None, M: torch.Tensor | None = None):
        self.kind, self.n, self.device = kind, n, torch.device(device)
        self._keep = (handle, X, M)
        o = OperatorT()
        o.kind, o.p = kind, int(p)
        o.h = handle.ptr if handle is not None else None
        if X is not None:
            o.X = X.data_ptr()
            o.n, o.ld_x, o.d = X.shape[0], X.stride(0), X.shape[1]
        if M is not None:
            o.M = M.data_ptr()
        self.c = o

    @classmethod
    def sorted(cls, h: Handle, p: int = 1) -> "Operator":
        return cls(OP_SORTED, h.n, torch.device("cuda", h.device), handle=h, p=p)

    @classmethod
    def even(cls, X: torch.Tensor, p: int) -> "Operator":
        X = _as_f32_2d(X, "X")
        if not X.is_cuda:
            raise ValueError("the even-p operator needs a CUDA X")
        return cls(OP_EVEN, X.shape[0], X.device, X=X, p=p)

    @classmethod
    def bilinear(cls, X: torch.Tensor, M: torch.Tensor) -> "Operator":
        X = _as_f32_2d(X, "X")
        M = torch.as_tensor(M, dtype=torch.float64, device=X.device).contiguous()
        if not X.is_cuda or tuple(M.shape) != (X.shape[1], X.shape[1]):
            raise ValueError("the bilinear operator needs a CUDA X and a d x d M")
        return cls(OP_BILINEAR, X.shape[0], X.device, X=X, M=M)


def _f64_dev(t, name, device):
    t = torch.as_tensor(t)
    if t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor (the dense steps run only in the library)")
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if t.device != device:
        raise ValueError(f"{name} must be on {device}")
    if t.dim() == 1:
        t = t.view(-1, 1)
    if t.stride(-1) != 1:
        t = t.contiguous()
    return t


def l1dm_gemm(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor | None = None, *,
              trans_a: bool = False, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """C = alpha op(A) B + beta C in fp64 on the tensor cores (device tensors, row-major)."""
    dev = A.device
    A, B = _f64_dev(A, "A", dev), _f64_dev(B, "B", dev)
    M = A.shape[1] if trans_a else A.shape[0]
    K = A.shape[0] if trans_a else A.shape[1]
    if B.shape[0] != K:
        raise ValueError(f"inner dimensions differ: op(A) is {M} x {K}, B is {tuple(B.shape)}")
    N = B.shape[1]
    if C is None:
        if beta != 0.0:
            raise ValueError("beta != 0 needs C")
        C = torch.empty((M, N), dtype=torch.float64, device=dev)
    C = _f64_dev(C, "C", dev)
    with torch.cuda.device(dev):
        _check(load_library().l1dm_gemm(1 if trans_a else 0, M, N, K, float(alpha), _ptr(A),
                                        A.stride(0), _ptr(B), B.stride(0), float(beta), _ptr(C),
                                        C.stride(0), _stream_of(C, stream)), "l1dm_gemm")
    return C


def l1dm_syevj(A: torch.Tensor, stream=None):
    """Symmetric eigen-decomposition (device Jacobi): returns (W, V), A V = V diag(W)."""
    dev = A.device
    A = _f64_dev(A, "A", dev)
    N = A.shape[0]
    if A.shape != (N, N):
        raise ValueError("A must be square")
    W = torch.empty(N, dtype=torch.float64, device=dev)
    V = torch.empty((N, N), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _check(load_library().l1dm_syevj(N, _ptr(A), A.stride(0), _ptr(W), _ptr(V), V.stride(0),
                                         _stream_of(A, stream)), "l1dm_syevj")
    return W, V


def l1dm_syev_topk(A: torch.Tensor, k: int, stream=None):
    """The k eigenpairs of largest |lambda| of a symmetric device matrix: (lam, V), A V = V lam."""
    dev = A.device
    A = _f64_dev(A, "A", dev)
    N = A.shape[0]
    lam = torch.empty(k, dtype=torch.float64, device=dev)
    V = torch.empty((N, k), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _check(load_library().l1dm_syev_topk(N, _ptr(A), A.stride(0), k, _ptr(lam), _ptr(V), k,
                                             _stream_of(A, stream)), "l1dm_syev_topk")
    return lam, V


def l1dm_op_apply(op: Operator, V: torch.Tensor, Y: torch.Tensor | None = None, stream=None):
    """A V for an fp64 block V (n x b) through the fp32 product (hi/lo split)."""
    squeeze = V.dim() == 1
    V = _f64_dev(V, "V", op.device)
    n, b = V.shape
    if n != op.n:
        raise ValueError(f"V has {n} rows, the operator {op.n}")
    if Y is None:
        Y = torch.empty((n, b), dtype=torch.float64, device=op.device)
    with torch.cuda.device(op.device):
        _check(load_library().l1dm_op_apply(ctypes.byref(op.c), _ptr(V), V.stride(0), b, _ptr(Y),
                                            Y.stride(0), _stream_of(V, stream)), "l1dm_op_apply")
    return Y.view(-1) if squeeze else Y


def l1dm_block_krylov(op: Operator, k: int, Pi: torch.Tensor, depth: int, stream=None):
    """Top-k |eigenvalues| (= singular values) of A by block Krylov from the start block Pi
    (n x b fp64); returns (sigma, lam, Z, info dict)."""
    Pi = _f64_dev(Pi, "Pi", op.device).contiguous()
    n, b = Pi.shape
    sigma = torch.empty(k, dtype=torch.float64, device=op.device)
    lam = torch.empty(k, dtype=torch.float64, device=op.device)
    Z = torch.empty((n, k), dtype=torch.float64, device=op.device)
    info = KrylovInfoT()
    with torch.cuda.device(op.device):
        _check(load_library().l1dm_block_krylov(ctypes.byref(op.c), k, b, depth, _ptr(Pi),
                                                _ptr(sigma), _ptr(lam), _ptr(Z), k,
                                                _stream_of(Pi, stream), ctypes.byref(info)),
               "l1dm_block_krylov")
    return sigma, lam, Z, {f: getattr(info, f) for f, _ in KrylovInfoT._fields_}


def l1dm_cg(op: Operator, b: torch.Tensor, *, tol: float = 1e-8, maxit: int = 500,
            normal_equations: bool = False, stream=None):
    """Conjugate gradients with device scalars; returns (x, info dict)."""
    b = _f64_dev(b, "b", op.device).reshape(-1).contiguous()
    x = torch.empty_like(b)
    info = CGInfoT()
    with torch.cuda.device(op.device):
        _check(load_library().l1dm_cg(ctypes.byref(op.c), _ptr(b), _ptr(x), float(tol), int(maxit),
                                      1 if normal_equations else 0, _stream_of(b, stream),
                                      ctypes.byref(info)), "l1dm_cg")
    return x, {f: getattr(info, f) for f, _ in CGInfoT._fields_}


class _DeviceView:
    """A zero-copy torch view of a device buffer the library hands to a callback."""

    def __init__(self, ptr: int, rows: int, cols: int, ld: int):
        self.__cuda_array_interface__ = {"shape": (rows, cols), "typestr": "<f8",
                                         "data": (int(ptr), False), "strides": (ld * 8, 8),
                                         "version": 2}


def device_view(ptr: int, rows: int, cols: int, ld: int, device) -> torch.Tensor:
    return torch.as_tensor(_DeviceView(ptr, rows, cols, ld), device=device)


def _callback(apply, n: int, device):
    """Wrap apply(V, Y, stream) -> None (torch views of the library's buffers; enqueue Y = A V on
    `stream`) as an l1dm_apply_fn.  Exceptions become a nonzero status (never cross the ABI)."""
    def cb(user, vptr, ldv, b, yptr, ldy, sptr):
        try:
            V = device_view(vptr, n, b, ldv, device)
            Y = device_view(yptr, n, b, ldy, device)
            st = torch.cuda.ExternalStream(sptr, device=device) if sptr else \
                torch.cuda.default_stream(device)
            with torch.cuda.stream(st):
                apply(V, Y, st)
            return 0
        except Exception:  # noqa: BLE001 — reported as a status through the C ABI
            import traceback
            traceback.print_exc()
            return -4
    return APPLY_FN(cb)


def l1dm_block_krylov_cb(n: int, apply, k: int, Pi: torch.Tensor, depth: int, stream=None):
    """Block Krylov with a caller-supplied product apply(V, Y, stream) (Y = A V, fp64 n x b
    views): every dense step in the library; returns (sigma, lam, Z, info dict)."""
    device = Pi.device
    Pi = _f64_dev(Pi, "Pi", device).contiguous()
    b = Pi.shape[1]
    sigma = torch.empty(k, dtype=torch.float64, device=device)
    lam = torch.empty(k, dtype=torch.float64, device=device)
    Z = torch.empty((n, k), dtype=torch.float64, device=device)
    info = KrylovInfoT()
    fn = _callback(apply, n, device)
    with torch.cuda.device(device):
        _check(load_library().l1dm_block_krylov_cb(n, fn, None, k, b, depth, _ptr(Pi), _ptr(sigma),
                                                   _ptr(lam), _ptr(Z), k, _stream_of(Pi, stream),
                                                   ctypes.byref(info)), "l1dm_block_krylov_cb")
    return sigma, lam, Z, {f: getattr(info, f) for f, _ in KrylovInfoT._fields_}


def l1dm_cg_cb(n: int, apply, b: torch.Tensor, *, tol: float = 1e-8, maxit: int = 500,
               normal_equations: bool = False, stream=None):
    """CG with a caller-supplied product apply(V, Y, stream); returns (x, info dict)."""
    device = b.device
    b = _f64_dev(b, "b", device).reshape(-1).contiguous()
    x = torch.empty_like(b)
    info = CGInfoT()
    fn = _callback(apply, n, device)
    with torch.cuda.device(device):
        _check(load_library().l1dm_cg_cb(n, fn, None, _ptr(b), _ptr(x), float(tol), int(maxit),
                                         1 if normal_equations else 0, _stream_of(b, stream),
                                         ctypes.byref(info)), "l1dm_cg_cb")
    return x, {f: getattr(info, f) for f, _ in CGInfoT._fields_}
