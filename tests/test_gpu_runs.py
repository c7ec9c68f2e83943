"""Runs mode (tie-heavy data: every coordinate <= 256 distinct values; include/l1dm.h
L1DM_MODE_RUNS) against the oracle.  Integer data must be bit-exact (HIST
oracle); float data with few distinct values meets the 1e-9 bar against brute force."""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_15114_b200 as l1
from conftest import col_rel_l2
from gpu_util import gpu_matvec

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.mark.parametrize("n,d,m", [(2, 1, 1), (1000, 3, 1), (40000, 12, 16), (5001, 4, 3),
                                   (3000, 5, 17), (2500, 2, 40), (1500, 3, 66), (1200, 2, 71),
                                   (777, 9, 2),
                                   # the expansion's run-id loop: 16-, 8- and 4-wide steps
                                   # with 4-wide and single remainders, narrow and wide shards
                                   (8000, 3, 66), (9000, 14, 8), (4500, 28, 4), (4500, 29, 4),
                                   (4097, 1, 4), (5000, 6, 16), (4100, 12, 12)])
def test_runs_integer_exact(n, d, m):
    rng = np.random.default_rng(n + 7 * m)
    X = rng.integers(0, 256, size=(n, d)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(n, m)).astype(np.float32)
    want = oracle.hist(X, Z, M=255).astype(np.float64)
    assert np.array_equal(gpu_matvec(X, Z, mode="runs"), want)
    assert np.array_equal(gpu_matvec(X, Z), want)                    # auto picks runs


@pytest.mark.parametrize("m", [2, 16, 33])
def test_runs_staged_expand_still_exact(m, monkeypatch):
    """The shared-memory-staged expansion (L1DM_RUNS_GATHER=0) stays correct; run in a fresh
    process so the environment switch takes effect."""
    import subprocess
    import sys
    code = (
        "import numpy as np, oracle, sys; sys.path.insert(0, 'tests');"
        "from gpu_util import gpu_matvec;"
        f"rng = np.random.default_rng({m});"
        "X = rng.integers(0, 256, size=(3000, 4)).astype(np.float32);"
        f"Z = rng.integers(-2, 3, size=(3000, {m})).astype(np.float32);"
        "w = oracle.hist(X, Z, M=255).astype(np.float64);"
        "assert np.array_equal(gpu_matvec(X, Z, mode='runs'), w)")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, L1DM_RUNS_GATHER="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def test_runs_float_values_and_constant_coordinate():
    rng = np.random.default_rng(3)
    n, d, m = 6000, 5, 6
    table = rng.standard_normal((d, 9)).astype(np.float32)           # 9 distinct values / coord
    X = table[np.arange(d)[None, :], rng.integers(0, 9, size=(n, d))]
    X[:, 2] = 1.25                                                   # one run
    Z = rng.standard_normal((n, m)).astype(np.float32)
    Yr = oracle.brute(X, Z)
    for mode in ("runs", "gather", "scatter"):
        assert col_rel_l2(gpu_matvec(X, Z, mode=mode), Yr) <= TOL, mode


def test_runs_unavailable_for_many_distinct_values():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((2000, 3)).astype(np.float32)           # ~2000 distinct per coord
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    with pytest.raises(l1.L1dmError):
        l1.l1dm_set_query_mode(h, "runs")
    l1.l1dm_free(h)


def test_runs_shards_and_pipelined_blocks():
    rng = np.random.default_rng(5)
    X = rng.integers(0, 40, size=(7001, 6)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(7001, 5)).astype(np.float32)
    whole = oracle.hist(X, Z, M=39).astype(np.float64)
    parts = [gpu_matvec(X, Z, a, b, mode="runs") for a, b in [(0, 2), (2, 6)]]
    assert np.array_equal(sum(parts), whole)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    l1.l1dm_set_query_mode(h, "runs")
    Y = torch.full((7001, 5), float("nan"), dtype=torch.float64, device="cuda")
    evs = [torch.cuda.Event() for _ in range(3)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    l1.l1dm_matvec_pipelined(h, torch.from_numpy(Z).cuda(), Y, evs, stream=side)
    for (i0, i1), ev in zip(l1.point_blocks(7001, 3), evs):
        ev.synchronize()
        assert np.array_equal(Y[i0:i1].cpu().numpy(), whole[i0:i1])
    l1.l1dm_sync(h)
    l1.l1dm_free(h)


def test_query_strategy_reports_the_planner_choice():
    """l1dm_query_strategy: runs on <= 256 distinct values (AUTO/RUNS), else the planner's
    gather/scatter choice under the handle's mode."""
    rng = np.random.default_rng(21)
    Xi = torch.from_numpy(rng.integers(0, 50, size=(3000, 4)).astype(np.float32)).cuda()
    h = l1.l1dm_prepare(Xi)
    try:
        assert l1.l1dm_query_strategy(h, 8) == "runs"
        l1.l1dm_set_query_mode(h, "gather")
        assert l1.l1dm_query_strategy(h, 8) == "gather"
        l1.l1dm_set_query_mode(h, "scatter")
        assert l1.l1dm_query_strategy(h, 8) == "scatter"
    finally:
        l1.l1dm_free(h)
    Xf = torch.from_numpy(rng.standard_normal((1 << 17, 3)).astype(np.float32)).cuda()
    h = l1.l1dm_prepare(Xf)
    try:
        assert l1.l1dm_query_strategy(h, 16) == "scatter"  # n >= 2^17, a block fits L2
        with pytest.raises(l1.L1dmError):
            l1.l1dm_set_query_mode(h, "runs")  # > 256 distinct values: no runs tables
    finally:
        l1.l1dm_free(h)
