"""The query planner (pure host function exported as l1dm_plan): tile/segment/chunk sizes."""
import pytest

import paper_2210_15114_b200 as l1

L2 = 126 << 20


@pytest.mark.parametrize("m,vec,lpr", [(1, 1, 1), (2, 2, 1), (3, 1, 4), (4, 4, 1), (5, 1, 8),
                                       (8, 4, 2), (16, 4, 4), (31, 1, 32), (32, 4, 8),
                                       (64, 4, 16), (65, 1, 32), (128, 4, 16), (6, 2, 4)])
def test_lane_mapping(m, vec, lpr):
    p = l1.l1dm_plan(1 << 20, 64, m, L2, 64 << 30)
    assert (p["vec"], p["lanes_per_row"]) == (vec, lpr)
    assert p["mb"] == vec * lpr
    assert p["col_blocks"] == -(-m // p["mb"])
    assert p["rows_per_tile"] == 8 * (32 // lpr) * 8
    assert p["tiles_per_segment"] == -(-(1 << 20) // p["rows_per_tile"])


def test_small_problem_is_l2_resident_and_chunked():
    p = l1.l1dm_plan(1 << 20, 64, 1, L2, 64 << 30)
    assert p["l2_resident"] == 1
    assert p["kc"] * (1 << 20) * 8 <= 0.4 * L2
    assert p["chunks"] == -(-64 // p["kc"])


def test_large_problem_uses_hbm_workspace():
    p = l1.l1dm_plan(1 << 20, 128, 64, L2, 100 << 30)
    assert p["l2_resident"] == 0
    assert p["kc"] == 128 and p["chunks"] == 1
    p = l1.l1dm_plan(1 << 24, 128, 32, L2, 64 << 30)
    assert p["kc"] == 15 and p["chunks"] == 9
    assert p["workspace_bytes"] <= 64 << 30


def test_workspace_limit_forces_chunks_and_minimum_one_coordinate():
    p = l1.l1dm_plan(100000, 10, 64, L2, 1)
    assert p["kc"] == 1 and p["chunks"] == 10


def test_invalid_sizes():
    for bad in [(0, 1, 1), (1, 0, 1), (1, 1, 0)]:
        with pytest.raises(l1.L1dmError):
            l1.l1dm_plan(*bad, L2, 0)
