"""Query parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): max over columns of the relative l2 error <= 1e-9 for float
data; bit-exact for integer data (every partial sum is an integer < 2^53)."""
from dataclasses import replace

import numpy as np
import pytest
import torch

import oracle
import paper_2210_15114_b200 as l1
from conftest import GOLDEN, col_rel_l2, load_golden, q12_rows
from gpu_util import gpu_matvec
from paper_2210_15114_b200 import workloads as wl

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.mark.parametrize("name", GOLDEN)
def test_golden(name):
    X, Z, Y = load_golden(name)
    assert np.array_equal(gpu_matvec(X, Z), Y)
    assert np.array_equal(gpu_matvec(X, Z, host=True), Y)


# m values exercise every lane mapping (vec 1/2/4, lanes per row 1..32, >1 column block);
# n values span several scan tiles (2048 rows at m=1 ... 64 rows at m=31) plus ragged tails.
CASES = [(1, 1, 1), (2, 1, 3), (3, 2, 2), (100, 3, 1), (2049, 2, 1), (4097, 3, 2), (5000, 4, 3),
         (1000, 5, 4), (3001, 3, 5), (700, 2, 8), (1029, 3, 16), (333, 2, 31), (777, 2, 32),
         (1100, 3, 64), (200, 2, 65), (513, 2, 128), (257, 3, 6), (6000, 1, 12)]


@pytest.mark.parametrize("n,d,m", CASES)
def test_random_float_vs_brute(n, d, m):
    rng = np.random.default_rng(n * 1000 + d * 10 + m)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Z = rng.standard_normal((n, m)).astype(np.float32)
    Yg = gpu_matvec(X, Z)
    Yr = oracle.brute(X, Z)
    assert col_rel_l2(Yg, Yr) <= TOL


@pytest.mark.parametrize("mode", ["gather", "scatter", "runs", "auto"])
@pytest.mark.parametrize("n,d,m", [(4099, 3, 1), (3000, 4, 4), (2500, 2, 7), (1500, 3, 32)])
def test_integer_ties_exact(n, d, m, mode):
    rng = np.random.default_rng(7 * n + m)
    X = rng.integers(0, 5, size=(n, d)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(n, m)).astype(np.float32)
    Yg = gpu_matvec(X, Z, mode=mode)
    assert np.array_equal(Yg, oracle.hist(X, Z, M=4).astype(np.float64))


def test_degenerate_cases():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((300, 3)).astype(np.float32)
    Z = rng.standard_normal((300, 2)).astype(np.float32)
    assert np.all(gpu_matvec(X, np.zeros_like(Z)) == 0)                       # z = 0
    # equal points: A = 0.  The U-form's g - h_i S cancels only to rounding, so bound |y_i|
    # against its natural scale max_j D_ij * sum_j |z_j| <= (sum_k 2 max|x_k|) * ||z||_1.
    Xe = np.tile(X[:1], (300, 1))
    Ye = gpu_matvec(Xe, Z)
    scale = 2 * np.abs(Xe).max(0).sum() * np.abs(Z).sum(0)
    assert np.all(np.abs(Ye) <= 1e-12 * scale)
    assert np.all(gpu_matvec(X[:1], Z[:1]) == 0)                              # n = 1
    E = np.eye(300, dtype=np.float32)[:, :64]
    A = gpu_matvec(X, E)
    assert np.all(np.abs(A[np.arange(64), np.arange(64)]) <= 1e-12 * np.abs(A).max())
    D = np.abs(X[:, None, :].astype(np.float64) - X[None, :64, :].astype(np.float64)).sum(-1)
    assert np.allclose(A, D, rtol=1e-12, atol=1e-12)                          # A e_j = column j


def test_symmetry_linearity_on_gpu():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((20000, 6)).astype(np.float32)
    Z = rng.standard_normal((20000, 2)).astype(np.float32)
    Y = gpu_matvec(X, Z)
    a = float(Z[:, 0].astype(np.float64) @ Y[:, 1])
    b = float(Z[:, 1].astype(np.float64) @ Y[:, 0])
    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b))


def test_strided_query_and_host_pointers():
    rng = np.random.default_rng(11)
    X = rng.standard_normal((3000, 4)).astype(np.float32)
    Zw = torch.from_numpy(rng.standard_normal((3000, 9)).astype(np.float32))
    Z = Zw[:, 1:6]                      # ld_z = 9 > m = 5, misaligned base
    Yr = oracle.brute(X, Z.contiguous().numpy())
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    Yg = l1.l1dm_matvec(h, Zw.cuda()[:, 1:6])
    torch.cuda.synchronize()
    assert col_rel_l2(Yg.cpu().numpy(), Yr) <= TOL
    Yh = l1.l1dm_matvec(h, Z.contiguous().numpy())       # host in, host out
    assert col_rel_l2(Yh.numpy(), Yr) <= TOL
    l1.l1dm_free(h)


@pytest.mark.parametrize("m", [1, 4, 32])
def test_chunked_workspace_matches(m):
    rng = np.random.default_rng(m)
    X = rng.standard_normal((5000, 7)).astype(np.float32)
    Z = rng.standard_normal((5000, m)).astype(np.float32)
    Yr = oracle.brute(X, Z)
    Y1 = gpu_matvec(X, Z, ws_limit=1)     # one coordinate per chunk: Y read-modify-write path
    assert col_rel_l2(Y1, Yr) <= TOL


def test_coordinate_shards_sum_to_whole():
    rng = np.random.default_rng(15)
    X = rng.integers(0, 9, size=(4000, 7)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(4000, 3)).astype(np.float32)
    parts = [gpu_matvec(X, Z, a, b, mode="gather") for a, b in [(0, 2), (2, 3), (3, 7)]]
    whole = oracle.hist(X, Z, M=8).astype(np.float64)
    assert np.array_equal(sum(parts), whole)
    assert np.array_equal(parts[1], oracle.hist(X[:, 2:3], Z, M=8).astype(np.float64))


def test_repeated_queries_same_handle():
    rng = np.random.default_rng(21)
    X = rng.standard_normal((9000, 5)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    for m in (1, 8, 3, 8, 1):
        Z = rng.standard_normal((9000, m)).astype(np.float32)
        Y = l1.l1dm_matvec(h, torch.from_numpy(Z).cuda())
        torch.cuda.synchronize()
        assert col_rel_l2(Y.cpu().numpy(), oracle.brute(X, Z)) <= TOL
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


# ---- the five BASELINE.json workloads, value structure at reduced n, vs the oracle ----
@pytest.mark.parametrize("name,n", [("c1", 2048), ("c2", 30000), ("c3", 6000), ("c4", 20000),
                                    ("c5", 40000), ("ctx1", 50000), ("ctx2", 5000),
                                    ("ctx3", 30000)])
def test_workload_reduced(name, n):
    w = wl.workload(name, n=n)
    X = wl.make_points(w, "cuda")
    Z = wl.make_query(w, 0, "cuda")
    Yg = gpu_matvec(X, Z)
    Xh, Zh = X.cpu().numpy(), Z.cpu().numpy()
    if name in ("c5", "ctx2"):  # integer coordinates: the HIST oracle (ctx2: fp32 z, 1e-9)
        want = oracle.hist(Xh, Zh, M=255).astype(np.float64) if name == "c5" else None
        if want is not None:
            assert np.array_equal(Yg, want)
        else:
            assert col_rel_l2(Yg, oracle.sort_based(Xh, Zh)) <= TOL
    elif name == "c1":
        assert col_rel_l2(Yg, oracle.brute(Xh, Zh)) <= TOL
    else:
        assert col_rel_l2(Yg, oracle.sort_based(Xh, Zh)) <= TOL


# ---- Q12: full BASELINE.json sizes, in the bench's launch configuration, on sampled rows ----
@pytest.mark.slow
@pytest.mark.parametrize("name,mode", [("c1", "auto"), ("c2", "auto"), ("c3", "auto"),
                                       ("c4", "auto"), ("c5", "auto"), ("c3", "gather"),
                                       ("c2", "gather"), ("c5", "gather"), ("c5", "scatter")])
def test_workload_full_size_sampled(name, mode):
    """SURVEY §8(c) SAMPLE mode (Q12; the definition P:149/P:171 at full n): auto is the bench's
    launch configuration (c2, c3: scatter; c4: gather; c5: runs).  Three back-to-back queries
    on one handle (recycled workspace: tile totals, Yt/Zt blocks, U, look-back epochs), each
    checked on SURVEY's rows: 64 seeded random rows + {0, n-1, argmin h, argmax h}."""
    w = wl.workload(name)
    wf = replace(w, fresh_queries=True)  # three different Z blocks, also for fixed-Pi c3
    X = wl.make_points(w, "cuda")
    h = l1.l1dm_prepare(X)
    l1.l1dm_set_query_mode(h, mode)
    Xh = X.cpu().numpy()
    rows = q12_rows(Xh)
    rows_d = torch.from_numpy(rows).cuda()
    Zs, got = [], []
    Y = torch.empty((w.n, w.m), dtype=torch.float64, device="cuda")
    for t in range(3):
        Z = wl.make_query(wf, t, "cuda")
        l1.l1dm_matvec(h, Z, Y)
        got.append(Y[rows_d].cpu().numpy())   # stream-ordered after the query
        Zs.append(Z.cpu().numpy())
    torch.cuda.synchronize()
    l1.l1dm_sync(h)
    del Y, X
    l1.l1dm_free(h)
    # one oracle pass over the three blocks side by side (m independent matvecs)
    Yr = oracle.rows(Xh, np.concatenate(Zs, axis=1), rows)
    for t in range(3):
        want = Yr[:, t * w.m:(t + 1) * w.m]
        if name == "c5":
            assert np.array_equal(got[t], want), f"query {t}"   # integers < 2^53: exact
        else:
            assert col_rel_l2(got[t], want) <= TOL, f"query {t}"


@pytest.mark.parametrize("m,blocks", [(1, 3), (4, 5), (64, 4)])
def test_pipelined_point_blocks(m, blocks):
    """l1dm_matvec_pipelined: same Y, and each block's event fires once its rows are final."""
    rng = np.random.default_rng(40 + m)
    X = rng.standard_normal((7001, 5)).astype(np.float32)
    Z = rng.standard_normal((7001, m)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    Zd = torch.from_numpy(Z).cuda()
    Y = torch.full((7001, m), float("nan"), dtype=torch.float64, device="cuda")
    evs = [torch.cuda.Event() for _ in range(blocks)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    l1.l1dm_matvec_pipelined(h, Zd, Y, evs, stream=side)
    ranges = l1.point_blocks(7001, blocks)
    assert ranges[0][0] == 0 and ranges[-1][1] == 7001
    Yr = oracle.brute(X, Z)
    for (i0, i1), ev in zip(ranges, evs):
        ev.synchronize()
        assert col_rel_l2(Y[i0:i1].cpu().numpy(), Yr[i0:i1]) <= TOL
    torch.cuda.synchronize()
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


@pytest.mark.parametrize("n", [1, 2, 3, 31, 4095, 4097, 9000])
def test_single_column_paths_small_and_ragged(n):
    """m = 1: the reduce-then-scan path (scatter-add into Y), strided Y."""
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 4)).astype(np.float32)
    Z = rng.standard_normal((n, 1)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    # the planner chooses scatter for m = 1 when Y fits L2; L1DM_SCATTER overrides it (read
    # once per process by the library, so the non-scatter case runs in a subprocess below)
    Yw = torch.full((n, 3), float("nan"), dtype=torch.float64, device="cuda")
    Y = Yw[:, 1:2]                                   # ld_y = 3 > m = 1
    lib = l1.load_library()
    import ctypes
    rc = lib.l1dm_matvec_ex(h.ptr, ctypes.c_void_p(torch.from_numpy(Z).cuda().data_ptr()), 1, 1,
                            ctypes.c_void_p(Y.data_ptr()), 3,
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    l1.l1dm_sync(h)
    Yr = oracle.brute(X, Z)
    if n == 1:
        assert Yw[0, 1].item() == 0.0
    else:
        assert col_rel_l2(Y.cpu().numpy(), Yr) <= TOL
    assert torch.isnan(Yw[:, 0]).all() and torch.isnan(Yw[:, 2]).all()   # ld_y respected
    l1.l1dm_free(h)


def test_scatter_mode_host_pointers_and_plan():
    rng = np.random.default_rng(77)
    X = rng.integers(0, 6, size=(20000, 3)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(20000, 1)).astype(np.float32)
    p = l1.l1dm_plan(20000, 3, 1)
    assert p["scatter"] == 1
    h = l1.l1dm_prepare(X)                           # host X
    l1.l1dm_set_query_mode(h, "scatter")            # (integer data would pick runs mode)
    Y = l1.l1dm_matvec(h, Z)                         # host Z, host Y
    assert np.array_equal(Y.numpy(), oracle.hist(X, Z, M=5).astype(np.float64))
    l1.l1dm_free(h)


def test_more_coordinates_than_one_chunk_exactly():
    """Integer data across several chunks (workspace limit) stays bit-exact."""
    rng = np.random.default_rng(78)
    X = rng.integers(0, 256, size=(30000, 9)).astype(np.float32)
    Z = (2 * rng.integers(0, 2, size=(30000, 16)) - 1).astype(np.float32)
    Yg = gpu_matvec(X, Z, ws_limit=3 * 30000 * 16 * 8, mode="gather")
    assert np.array_equal(Yg, oracle.hist(X, Z, M=255).astype(np.float64))


def test_single_column_gather_mode_subprocess():
    """m = 1 without scatter (U + rank gather), forced by L1DM_SCATTER=0 in a fresh process."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['.', 'tests']; import test_gpu_parity as t;"
            "[t.test_single_column_paths_small_and_ragged(n) for n in (1, 2, 3, 31, 4097, 9000)];"
            "t.test_random_float_vs_brute(2049, 2, 1); print('ok')")
    env = dict(os.environ, L1DM_SCATTER="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_pinned_host_pipeline_async_queries():
    """Pinned host Z and Y: asynchronous calls with overlapped copies; results after l1dm_sync
    equal the oracle for every query (staging slots alternate, Y buffers distinct)."""
    rng = np.random.default_rng(123)
    X = rng.standard_normal((5000, 6)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    Zs = [torch.from_numpy(rng.standard_normal((5000, 7)).astype(np.float32)).pin_memory()
          for _ in range(5)]
    Ys = [torch.empty((5000, 7), dtype=torch.float64).pin_memory() for _ in range(5)]
    for Z, Y in zip(Zs, Ys):
        l1.l1dm_matvec(h, Z, Y, block=False)
    l1.l1dm_sync(h)
    for Z, Y in zip(Zs, Ys):
        assert col_rel_l2(Y.numpy(), oracle.brute(X, Z.numpy())) <= TOL
    Yb = l1.l1dm_matvec(h, Zs[0], torch.empty((5000, 7), dtype=torch.float64).pin_memory())
    assert col_rel_l2(Yb.numpy(), oracle.brute(X, Zs[0].numpy())) <= TOL   # block=True default
    l1.l1dm_free(h)


def test_handle_utilities_and_block_cache():
    """l1dm_shape / l1dm_workspace_bytes on a sharded handle; handles recycling each other's
    device blocks through the library's cache, then l1dm_release_cached, stay exact."""
    import ctypes
    rng = np.random.default_rng(77)
    X = rng.integers(0, 9, size=(3000, 6)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(3000, 5)).astype(np.float32)
    want = oracle.brute(X, Z)
    Xt, Zt = torch.from_numpy(X).cuda(), torch.from_numpy(Z).cuda()
    lib = l1.load_library()
    for rep in range(3):
        h = l1.l1dm_prepare(Xt, 1, 5)
        vals = [ctypes.c_int64() for _ in range(4)]
        assert lib.l1dm_shape(h.ptr, *[ctypes.byref(v) for v in vals]) == 0
        assert [v.value for v in vals] == [3000, 4, 1, 5]  # n, d_local, k_begin, k_end
        l1.l1dm_set_query_mode(h, "gather")
        assert l1.l1dm_workspace_bytes(h, 5) >= 3000 * 4 * 5 * 8  # U of the shard
        l1.l1dm_free(h)
        h = l1.l1dm_prepare(Xt)
        Y = l1.l1dm_matvec(h, Zt)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().numpy(), want), rep
        l1.l1dm_free(h)
        if rep == 1:
            l1.l1dm_release_cached()


def test_empty_and_invalid_sizes_rejected():
    """SURVEY A9 / include/l1dm.h: n, d, m >= 1 — empty inputs are rejected with EINVAL (no
    kernel runs), an empty coordinate range too; n = 1 is the smallest valid case (Y = 0)."""
    with pytest.raises(l1.L1dmError) as e:
        l1.l1dm_prepare(torch.zeros((0, 3), device="cuda"))
    assert e.value.name == "L1DM_EINVAL"
    with pytest.raises(l1.L1dmError) as e:
        l1.l1dm_prepare(torch.zeros((5, 0), device="cuda"))
    assert e.value.name == "L1DM_EINVAL"
    X = torch.rand((7, 3), device="cuda")
    with pytest.raises(l1.L1dmError) as e:
        l1.l1dm_prepare(X, 2, 2)
    assert e.value.name == "L1DM_EINVAL"
    h = l1.l1dm_prepare(X)
    with pytest.raises((l1.L1dmError, ValueError)):
        l1.l1dm_matvec(h, torch.zeros((7, 0), device="cuda"))
    with pytest.raises((l1.L1dmError, ValueError)):
        l1.l1dm_matvec(h, torch.zeros((6, 2), device="cuda"))   # wrong number of rows
    l1.l1dm_free(h)
    h1 = l1.l1dm_prepare(torch.tensor([[1.5, -2.0]], device="cuda"))
    Y = l1.l1dm_matvec(h1, torch.tensor([[3.0]], device="cuda"))
    torch.cuda.synchronize()
    assert float(Y.abs().max()) == 0.0
    l1.l1dm_free(h1)
