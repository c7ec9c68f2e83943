"""CPU oracle for Y = A·Z with A_ij = ||x_i - x_j||_1 (Alg. 1-2).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_2210_15114_b200) never imports it and shares no code with it.

The arithmetic lives in l1dm_oracle.c (plain C, long double accumulation);
this module only compiles it with gcc and marshals numpy arrays through ctypes.
Every function is pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "l1dm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, EINVAL, ENOMEM, ENOTINT = 0, -1, -2, -3


def build(force: bool = False) -> str:
    """Compile l1dm_oracle.c into oracle/liboracle.so (no fast-math: IEEE semantics kept)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.oracle_brute.argtypes = [vp, i64, i64, vp, i64, vp, i32]
        lib.oracle_rows.argtypes = [vp, i64, i64, vp, i64, vp, i64, vp, i32]
        lib.oracle_alg1.argtypes = [vp, i64, i64, vp, vp, i32]
        lib.oracle_alg2.argtypes = [vp, i64, i64, vp, vp, i64, vp, i32]
        lib.oracle_alg2_range.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, vp, i32]
        lib.oracle_hist.argtypes = [vp, i64, i64, vp, i64, i64, vp, i32]
        lib.oracle_num_threads.argtypes = [i32]
        lib.oracle_brute_lp.argtypes = [vp, i64, i64, vp, i64, i32, vp, i32]
        lib.oracle_lp_sorted.argtypes = [vp, i64, i64, vp, vp, i64, i32, vp, i32]
        lib.oracle_brute_tv.argtypes = [vp, i64, i64, vp, i64, vp, i32]
        lib.oracle_rows_lp.argtypes = [vp, i64, i64, vp, i64, i32, vp, i64, vp, i32]
        lib.oracle_lp_even.argtypes = [vp, i64, i64, vp, i64, i32, vp, i32]
        lib.oracle_brute_bilinear.argtypes = [vp, i64, i64, vp, vp, i64, vp, i32]
        lib.oracle_bilinear_alg.argtypes = [vp, i64, i64, vp, vp, i64, vp]
        lib.oracle_l2_embed.argtypes = [vp, i64, i64, vp, i64, vp]
        lib.oracle_brute_l2.argtypes = [vp, i64, i64, vp, i64, vp, i32]
        for f in (lib.oracle_brute, lib.oracle_rows, lib.oracle_alg1, lib.oracle_alg2,
                  lib.oracle_alg2_range, lib.oracle_hist, lib.oracle_num_threads,
                  lib.oracle_brute_lp, lib.oracle_lp_sorted, lib.oracle_brute_tv,
                  lib.oracle_rows_lp, lib.oracle_lp_even, lib.oracle_brute_bilinear,
                  lib.oracle_bilinear_alg, lib.oracle_l2_embed, lib.oracle_brute_l2):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _as2d(Z, n):
    Z = _f32(Z)
    if Z.ndim == 1:
        Z = Z.reshape(n, 1)
    return Z


def _check(rc, what):
    if rc != OK:
        raise ValueError(f"{what} failed with status {rc}")


def num_threads(nthreads: int = 0) -> int:
    return _load().oracle_num_threads(nthreads)


def brute(X, Z, nthreads: int = 0) -> np.ndarray:
    """Definition: Y[i,c] = sum_j Z[j,c] * ||x_i - x_j||_1. O(n^2 (d+m))."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_brute(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], _ptr(Y), nthreads), "brute")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def rows(X, Z, row_ids, nthreads: int = 0) -> np.ndarray:
    """Definition evaluated for the listed rows only: returns len(row_ids) x m."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    r = np.ascontiguousarray(row_ids, dtype=np.int64)
    Y = np.empty((r.shape[0], Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_rows(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], _ptr(r), r.shape[0],
                               _ptr(Y), nthreads), "rows")
    return Y


def alg1(X, nthreads: int = 0):
    """Alg. 1: per coordinate the sorted values T_i and the order pi^i.

    Returns (T, order), each d x n (coordinate-major); ties ordered by point index."""
    X = _f32(X)
    n, d = X.shape
    T = np.empty((d, n), dtype=np.float32)
    order = np.empty((d, n), dtype=np.uint32)
    _check(_load().oracle_alg1(_ptr(X), n, d, _ptr(T), _ptr(order), nthreads), "alg1")
    return T, order


def alg2(X, order, Z, nthreads: int = 0) -> np.ndarray:
    """Alg. 2 literally, one column of Z at a time (Lemma matrixmult)."""
    X = _f32(X)
    n, d = X.shape
    order = np.ascontiguousarray(order, dtype=np.uint32)
    assert order.shape == (d, n)
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_alg2(_ptr(X), n, d, _ptr(order), _ptr(Z2), Z2.shape[1], _ptr(Y),
                               nthreads), "alg2")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def alg2_range(X, order, k0, k1, Z, nthreads: int = 0) -> np.ndarray:
    """Alg. 2 over the coordinate slice [k0, k1) only: that slice's share of A·Z."""
    X = _f32(X)
    n, d = X.shape
    order = np.ascontiguousarray(order, dtype=np.uint32)
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_alg2_range(_ptr(X), n, d, _ptr(order), k0, k1, _ptr(Z2), Z2.shape[1],
                                     _ptr(Y), nthreads), "alg2_range")
    return Y


def sort_based(X, Z, nthreads: int = 0) -> np.ndarray:
    """Alg. 1 then Alg. 2: the paper's method, run as written."""
    _, order = alg1(X, nthreads)
    return alg2(X, order, Z, nthreads)


def hist(X, Z, M: int = 255, nthreads: int = 0) -> np.ndarray:
    """Exact int64 evaluation for X in {0..M}^(n x d) and integer-valued Z."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.int64)
    _check(_load().oracle_hist(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], M, _ptr(Y), nthreads), "hist")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def brute_lp(X, Z, p: int, nthreads: int = 0) -> np.ndarray:
    """l_p^p definition: Y[i,c] = sum_j Z[j,c] sum_k |x_ik - x_jk|^p (Thm. odd_p)."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_brute_lp(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], int(p), _ptr(Y),
                                   nthreads), "brute_lp")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def rows_lp(X, Z, p: int, row_ids, nthreads: int = 0) -> np.ndarray:
    """l_p^p definition for the listed rows only: returns len(row_ids) x m."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    r = np.ascontiguousarray(row_ids, dtype=np.int64)
    Y = np.empty((r.shape[0], Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_rows_lp(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], int(p), _ptr(r),
                                  r.shape[0], _ptr(Y), nthreads), "rows_lp")
    return Y


def lp_sorted(X, Z, p: int, nthreads: int = 0) -> np.ndarray:
    """Odd p with Alg. 1's sort: SPEC S:150-158's construction in Alg. 2's shape."""
    X = _f32(X)
    n, d = X.shape
    _, order = alg1(X, nthreads)
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_lp_sorted(_ptr(X), n, d, _ptr(np.ascontiguousarray(order)), _ptr(Z2),
                                    Z2.shape[1], int(p), _ptr(Y), nthreads), "lp_sorted")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def brute_tv(X, Z, nthreads: int = 0) -> np.ndarray:
    """TV definition: Y[i,c] = sum_j Z[j,c] (1/2) sum_k |x_ik - x_jk| (Thm. tv)."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_brute_tv(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], _ptr(Y), nthreads),
           "brute_tv")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def lp_even(X, Z, p: int, nthreads: int = 0) -> np.ndarray:
    """Even p: Alg. "query_p_even" with SPEC S:140-146's corrections."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_lp_even(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], int(p), _ptr(Y),
                                  nthreads), "lp_even")
    return Y.reshape(-1) if np.ndim(Z) == 1 else Y


def brute_bilinear(X, M, Z, nthreads: int = 0) -> np.ndarray:
    """Thm. maha's form, the definition: Y[i,c] = sum_j Z[j,c] x_i^T M x_j."""
    X = _f32(X)
    n, d = X.shape
    M = np.ascontiguousarray(M, dtype=np.float64)
    assert M.shape == (d, d)
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_brute_bilinear(_ptr(X), n, d, _ptr(M), _ptr(Z2), Z2.shape[1], _ptr(Y),
                                         nthreads), "brute_bilinear")
    return Y


def bilinear_alg(X, M, Z) -> np.ndarray:
    """Algs. 7-8 step by step: S = [M x_j]_j, v = S y, z(k) = <x_k, v>."""
    X = _f32(X)
    n, d = X.shape
    M = np.ascontiguousarray(M, dtype=np.float64)
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_bilinear_alg(_ptr(X), n, d, _ptr(M), _ptr(Z2), Z2.shape[1], _ptr(Y)),
           "bilinear_alg")
    return Y


def l2_embed(X, G) -> np.ndarray:
    """Thm. l2embed: X' = X G^T / (beta k), beta = sqrt(2/pi), rounded to fp32."""
    X = _f32(X)
    G = _f32(G)
    n, d = X.shape
    k = G.shape[0]
    assert G.shape[1] == d
    Xp = np.empty((n, k), dtype=np.float32)
    _check(_load().oracle_l2_embed(_ptr(X), n, d, _ptr(G), k, _ptr(Xp)), "l2_embed")
    return Xp


def brute_l2(X, Z, nthreads: int = 0) -> np.ndarray:
    """The exact l2 distance product: Y[i,c] = sum_j Z[j,c] ||x_i - x_j||_2."""
    X = _f32(X)
    n, d = X.shape
    Z2 = _as2d(Z, n)
    Y = np.empty((n, Z2.shape[1]), dtype=np.float64)
    _check(_load().oracle_brute_l2(_ptr(X), n, d, _ptr(Z2), Z2.shape[1], _ptr(Y), nthreads),
           "brute_l2")
    return Y
