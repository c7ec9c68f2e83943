"""Scatter-mode query (L1DM_MODE_SCATTER: per column block, the scan adds 2U into an
L2-resident block accumulator with fp64 reductions; include/l1dm.h) against the CPU oracle.

The planner picks this mode for n >= 2^17 when a block fits L2, so small
parity cases force it per handle; the full-size c3 case runs it by default (bench config).
Bar as in test_gpu_parity.py: per-column relative l2 <= 1e-9 on float data, bit-exact on
integer data (every partial sum is an integer < 2^53)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_15114_b200 as l1
from conftest import col_rel_l2
from gpu_util import gpu_matvec

pytestmark = pytest.mark.gpu
TOL = 1e-9

# m spans block widths 2 / 4 / 8 and ragged last blocks; n spans the 1024-row tiles' edges.
# m = 1 runs the same single-pass kernel with one-column blocks (2048-row tiles).
CASES = [(1, 1, 2), (2, 1, 3), (3, 2, 2), (100, 3, 4), (1023, 2, 5), (1024, 3, 8), (1025, 2, 9),
         (2047, 3, 16), (3073, 4, 7), (5000, 2, 17), (700, 5, 64), (1500, 3, 65), (4097, 2, 3),
         (1, 1, 1), (2049, 3, 1), (5000, 4, 1)]


@pytest.mark.parametrize("n,d,m", CASES)
def test_scatter_random_float_vs_brute(n, d, m):
    rng = np.random.default_rng(n * 977 + d * 31 + m)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Z = rng.standard_normal((n, m)).astype(np.float32)
    Yr = oracle.brute(X, Z)
    Ys = gpu_matvec(X, Z, mode="scatter")
    if n == 1:
        assert np.all(Ys == 0)
    else:
        assert col_rel_l2(Ys, Yr) <= TOL


@pytest.mark.parametrize("n,d,m", [(4099, 3, 2), (3000, 4, 4), (2500, 2, 7), (1500, 3, 32),
                                   (4100, 3, 1)])
def test_scatter_integer_ties_exact(n, d, m):
    rng = np.random.default_rng(7 * n + m + 1)
    X = rng.integers(0, 5, size=(n, d)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(n, m)).astype(np.float32)
    assert np.array_equal(gpu_matvec(X, Z, mode="scatter"),
                          oracle.hist(X, Z, M=4).astype(np.float64))


def test_scatter_and_gather_agree_on_one_handle():
    """Switching the mode on a live handle reuses/reallocates the workspace correctly."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((6000, 5)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    for mode, m in [("scatter", 12), ("gather", 12), ("scatter", 3), ("auto", 12), ("scatter", 40)]:
        Z = rng.standard_normal((6000, m)).astype(np.float32)
        l1.l1dm_set_query_mode(h, mode)
        Y = l1.l1dm_matvec(h, torch.from_numpy(Z).cuda())
        torch.cuda.synchronize()
        assert col_rel_l2(Y.cpu().numpy(), oracle.brute(X, Z)) <= TOL, mode
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


def test_scatter_strided_and_host_pointers():
    rng = np.random.default_rng(12)
    X = rng.standard_normal((3000, 4)).astype(np.float32)
    Zw = torch.from_numpy(rng.standard_normal((3000, 13)).astype(np.float32))
    Yr = oracle.brute(X, Zw[:, 1:11].contiguous().numpy())
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    l1.l1dm_set_query_mode(h, "scatter")
    Yg = l1.l1dm_matvec(h, Zw.cuda()[:, 1:11])          # ld_z = 13, misaligned base
    torch.cuda.synchronize()
    assert col_rel_l2(Yg.cpu().numpy(), Yr) <= TOL
    Yh = l1.l1dm_matvec(h, Zw[:, 1:11].contiguous().numpy())   # host in, host out
    assert col_rel_l2(Yh.numpy(), Yr) <= TOL
    import ctypes                                         # strided Y (ld_y = 14 > m = 10)
    Yw = torch.full((3000, 14), float("nan"), dtype=torch.float64, device="cuda")
    Zc = Zw[:, 1:11].contiguous().cuda()
    rc = l1.load_library().l1dm_matvec_ex(
        h.ptr, ctypes.c_void_p(Zc.data_ptr()), 10, 10, ctypes.c_void_p(Yw[:, 2:].data_ptr()), 14,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    l1.l1dm_sync(h)
    assert col_rel_l2(Yw[:, 2:12].cpu().numpy(), Yr) <= TOL
    assert torch.isnan(Yw[:, :2]).all() and torch.isnan(Yw[:, 12:]).all()
    l1.l1dm_free(h)


@pytest.mark.parametrize("m,blocks", [(4, 5), (20, 3)])
def test_scatter_pipelined_point_blocks(m, blocks):
    rng = np.random.default_rng(90 + m)
    X = rng.standard_normal((7001, 5)).astype(np.float32)
    Z = rng.standard_normal((7001, m)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    l1.l1dm_set_query_mode(h, "scatter")
    Y = torch.full((7001, m), float("nan"), dtype=torch.float64, device="cuda")
    evs = [torch.cuda.Event() for _ in range(blocks)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    l1.l1dm_matvec_pipelined(h, torch.from_numpy(Z).cuda(), Y, evs, stream=side)
    Yr = oracle.brute(X, Z)
    for (i0, i1), ev in zip(l1.point_blocks(7001, blocks), evs):
        ev.synchronize()
        assert col_rel_l2(Y[i0:i1].cpu().numpy(), Yr[i0:i1]) <= TOL
    torch.cuda.synchronize()
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


def test_scatter_degenerate():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((300, 3)).astype(np.float32)
    Z = rng.standard_normal((300, 6)).astype(np.float32)
    assert np.all(gpu_matvec(X, np.zeros_like(Z), mode="scatter") == 0)
    E = np.eye(300, dtype=np.float32)[:, :16]
    A = gpu_matvec(X, E, mode="scatter")
    D = np.abs(X[:, None, :].astype(np.float64) - X[None, :16, :].astype(np.float64)).sum(-1)
    assert np.allclose(A, D, rtol=1e-12, atol=1e-12)                  # A e_j = column j


def test_scatter_sharded_coordinates_exact():
    rng = np.random.default_rng(16)
    X = rng.integers(0, 9, size=(4000, 7)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(4000, 10)).astype(np.float32)
    parts = [gpu_matvec(X, Z, a, b, mode="scatter") for a, b in [(0, 2), (2, 3), (3, 7)]]
    assert np.array_equal(sum(parts), oracle.hist(X, Z, M=8).astype(np.float64))


def test_scatter_wide_query():
    """m > 256 (more than 32 column blocks of the single-pass apply)."""
    rng = np.random.default_rng(300)
    X = rng.standard_normal((1500, 2)).astype(np.float32)
    Z = rng.standard_normal((1500, 300)).astype(np.float32)
    assert col_rel_l2(gpu_matvec(X, Z, mode="scatter"), oracle.brute(X, Z)) <= TOL


# the two-pass forms (tile totals from a reduce pass, then the apply), selected per process:
# L1DM_SCATTER_LB=0 with the reduce-all pass over full Z rows, and with one reduce per block
# (odd p: the per-block reduce, then the apply with the totals); L1DM_LB_NT=256: the single-pass
# apply with 1024-row tiles (default 512)
@pytest.mark.parametrize("env", [{"L1DM_SCATTER_LB": "0"},
                                 {"L1DM_SCATTER_LB": "0", "L1DM_REDUCE_ALL": "0"},
                                 {"L1DM_LB_NT": "256"}])
def test_scatter_variants_subprocess(env):
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['.', 'tests']; import test_gpu_scatter as t;"
            "[t.test_scatter_random_float_vs_brute(*c) for c in t.CASES];"
            "t.test_scatter_integer_ties_exact(3000, 4, 4); t.test_scatter_wide_query();"
            "t.test_scatter_bitwise_reproducible();"
            "import test_gpu_lp as lp;"
            "[lp.test_lp_random_float_vs_oracle(*c, p, 'scatter') for c in lp.CASES for p in (3, 5, 7)];"
            "[lp.test_lp_integer_ties_exact(p, 'scatter') for p in (3, 5)]; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_colblocks_output_and_unblock():
    """l1dm_matvec_colblocks: block cb of the column-block-major output is final when its event
    fires; l1dm_unblock gives back the row-major Y (ragged last block included)."""
    rng = np.random.default_rng(44)
    X = rng.standard_normal((5000, 4)).astype(np.float32)
    Z = rng.standard_normal((5000, 21)).astype(np.float32)
    Yr = oracle.brute(X, Z)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    l1.l1dm_set_query_mode(h, "scatter")
    scatter, mb, ncb = l1.binding.l1dm_query_layout(h, 21)
    assert scatter == 1 and ncb == -(-21 // mb)
    Yb = torch.full((ncb, 5000, mb), float("nan"), dtype=torch.float64, device="cuda")
    evs = [torch.cuda.Event() for _ in range(ncb)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    l1.binding.l1dm_matvec_colblocks(h, torch.from_numpy(Z).cuda(), Yb, evs, stream=side)
    for cb, ev in enumerate(evs):
        ev.synchronize()
        c0, c1 = cb * mb, min(21, cb * mb + mb)
        assert col_rel_l2(Yb[cb, :, :c1 - c0].cpu().numpy(), Yr[:, c0:c1]) <= TOL
    Y = torch.empty((5000, 21), dtype=torch.float64, device="cuda")
    l1.binding.l1dm_unblock(Yb, 21, Y, stream=side)
    side.synchronize()
    assert col_rel_l2(Y.cpu().numpy(), Yr) <= TOL
    l1.l1dm_set_query_mode(h, "gather")
    with pytest.raises(l1.L1dmError):
        l1.binding.l1dm_matvec_colblocks(h, torch.from_numpy(Z).cuda(), Yb, evs)
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


def _scatter_handle(X):
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    l1.l1dm_set_query_mode(h, "scatter")
    return h


def test_scatter_bitwise_reproducible():
    """m > 1 scatter accumulates in 64-bit fixed point (R16): the same query on the
    same handle gives the same Y bit for bit, whatever order the L2 reductions land in."""
    rng = np.random.default_rng(11)
    X = rng.standard_normal((150000, 12)).astype(np.float32)
    Z = torch.from_numpy(rng.standard_normal((150000, 24)).astype(np.float32)).cuda()
    h = _scatter_handle(X)
    Ys = [l1.l1dm_matvec(h, Z).cpu() for _ in range(4)]
    l1.l1dm_free(h)
    assert all(torch.equal(Ys[0], y) for y in Ys[1:])


@pytest.mark.parametrize("xscale,zscales", [(1.0, (1e12, 1.0, 1e-12, 0.0)),
                                             (1e-18, (1e-20, 1e-3, 1.0, 1e-20)),
                                             (1e18, (1e15, 1.0, 1e-15, 3.0))])
def test_scatter_columns_of_different_scales(xscale, zscales):
    """Each column gets its own fixed-point scale from its own |z| sum: a column 24 orders of
    magnitude below its neighbour, tiny and huge data all meet the 1e-9 bar; a zero column is
    exactly zero."""
    rng = np.random.default_rng(13)
    n, d = 3000, 4
    X = (rng.standard_normal((n, d)) * xscale).astype(np.float32)
    Z = np.stack([rng.standard_normal(n) * s for s in zscales] * 3, axis=1).astype(np.float32)
    h = _scatter_handle(X)
    Y = l1.l1dm_matvec(h, torch.from_numpy(Z).cuda()).cpu().numpy()
    l1.l1dm_free(h)
    Yr = oracle.brute(X, Z)
    for c in range(Z.shape[1]):
        if not Z[:, c].any():
            assert not Y[:, c].any()
        else:
            assert col_rel_l2(Y[:, c:c + 1], Yr[:, c:c + 1]) <= TOL, c


@pytest.mark.parametrize("m", [1, 5])
def test_scatter_nonfinite_z_column_is_nan(m):
    """A NaN / Inf in a column of Z is not hidden by the fixed-point accumulation: that column of
    Y comes out NaN (include/l1dm.h), the other columns are unaffected."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 3)).astype(np.float32)
    Z = rng.standard_normal((3000, m)).astype(np.float32)
    Zb = Z.copy()
    Zb[17, 0] = np.nan
    if m > 1:
        Zb[5, m - 1] = np.inf
    Y = gpu_matvec(X, Zb, mode="scatter")
    assert np.all(np.isnan(Y[:, 0]))
    if m > 1:
        assert not np.any(np.isfinite(Y[:, m - 1]))
        Yr = oracle.brute(X, Z)
        assert col_rel_l2(Y[:, 1:m - 1], Yr[:, 1:m - 1]) <= TOL
