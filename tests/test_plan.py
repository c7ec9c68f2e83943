"""The query planner (pure host function exported as l1dm_plan): tile/segment/chunk sizes."""
import pytest

import paper_2210_15114_b200 as l1

L2 = 126 << 20


def scan_items(lpr, vc):
    if lpr == 1 and vc == 1:
        return 8                       # the single-column kernel: 8 consecutive rows per thread
    budget = 65536 if lpr == 32 else 98304  # stage bytes per tile (l1dm_internal.h)
    it = (budget // (1024 * vc + 2048 // lpr)) // 4 * 4
    return min(it, 64)


# (m, gather floats per cp.async, lanes per row, columns per segment)
@pytest.mark.parametrize("m,vec,lpr,mb", [(1, 1, 1, 1), (2, 2, 2, 2), (3, 1, 4, 4), (4, 4, 4, 4),
                                          (5, 1, 8, 8), (8, 4, 8, 8), (16, 4, 16, 16),
                                          (31, 1, 32, 32), (32, 4, 32, 32), (64, 4, 32, 64),
                                          (65, 1, 32, 32), (128, 4, 32, 64), (6, 2, 8, 8),
                                          (34, 2, 32, 64)])
def test_lane_mapping(m, vec, lpr, mb):
    p = l1.l1dm_plan(1 << 20, 64, m, L2, 64 << 30, mode="gather")
    assert (p["vec"], p["lanes_per_row"], p["mb"]) == (vec, lpr, mb)
    assert p["col_blocks"] == -(-m // p["mb"])
    assert p["rows_per_tile"] == 8 * (32 // lpr) * scan_items(lpr, mb // lpr)
    assert p["tiles_per_segment"] == -(-(1 << 20) // p["rows_per_tile"])


def test_small_problem_is_l2_resident_and_chunked():
    p = l1.l1dm_plan(1 << 20, 64, 2, L2, 64 << 30, mode="gather")
    assert p["l2_resident"] == 1 and p["scatter"] == 0
    assert p["kc"] * (1 << 20) * 2 * 8 <= 0.4 * L2
    assert p["chunks"] == -(-64 // p["kc"])


def test_single_column_small_n_uses_scatter_mode():
    p = l1.l1dm_plan(1 << 20, 64, 1, L2, 64 << 30)
    assert p["scatter"] == 1 and p["chunks"] == 1 and p["kc"] == 64
    p = l1.l1dm_plan(1 << 24, 64, 1, L2, 64 << 30)   # Y (128 MiB) does not fit L2
    assert p["scatter"] == 0


def test_large_problem_uses_hbm_workspace():
    p = l1.l1dm_plan(1 << 20, 128, 64, L2, 100 << 30, mode="gather")
    assert p["l2_resident"] == 0
    assert p["kc"] == 128 and p["chunks"] == 1
    p = l1.l1dm_plan(1 << 24, 128, 32, L2, 64 << 30)
    assert p["kc"] == 15 and p["chunks"] == 9   # U per coordinate = 4 GiB (+ look-back state)
    assert p["workspace_bytes"] <= 64 << 30


def test_workspace_limit_forces_chunks_and_minimum_one_coordinate():
    p = l1.l1dm_plan(100000, 10, 64, L2, 1)
    assert p["kc"] == 1 and p["chunks"] == 10


def test_invalid_sizes():
    for bad in [(0, 1, 1), (1, 0, 1), (1, 1, 0)]:
        with pytest.raises(l1.L1dmError):
            l1.l1dm_plan(*bad, L2, 0)


# (n, m) -> expected (scatter, columns per block) under the measured crossovers
@pytest.mark.parametrize("n,m,scatter,mb", [
    (1 << 20, 64, 1, 8), (1 << 20, 16, 1, 8), (1 << 20, 5, 1, 8), (1 << 20, 3, 1, 4),
    (1 << 20, 2, 1, 2), (3 << 19, 16, 1, 8), (1 << 21, 16, 1, 4), (1 << 21, 64, 0, 64),
    (1 << 24, 32, 0, 32), ((1 << 17) - 1, 64, 0, 64), (1 << 17, 64, 1, 8)])
def test_scatter_plan_crossovers(n, m, scatter, mb):
    p = l1.l1dm_plan(n, 64, m, 132644864, 64 << 30)
    assert (p["scatter"], p["mb"]) == (scatter, mb)
    if scatter:
        assert p["col_blocks"] == -(-m // mb) and p["kc"] == 64 and p["chunks"] == 1
        assert p["rows_per_tile"] == 1024 and p["tiles_per_segment"] == -(-n // 1024)


def test_query_mode_overrides_the_crossover():
    assert l1.l1dm_plan(1 << 20, 64, 64, L2, 64 << 30, mode="gather")["scatter"] == 0
    p = l1.l1dm_plan(1 << 21, 64, 64, L2, 64 << 30, mode="scatter")
    assert p["scatter"] == 1 and p["mb"] == 4
    assert l1.l1dm_plan(1000, 4, 1, L2, 0, mode="scatter")["scatter"] == 1
    with pytest.raises(l1.L1dmError):
        l1.l1dm_plan(1000, 4, 1, L2, 0, mode=7)
