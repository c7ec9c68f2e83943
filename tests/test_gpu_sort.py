"""Prepare-stage parity (Alg. 1): the GPU radix sort tables against the oracle's
comparison sort, bit-exact (pin Q13).  Ties by index, -0.0 ordered as +0.0."""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def check_tables(X, k_begin=0, k_end=None):
    n, d = X.shape
    k_end = d if k_end is None else k_end
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda(), k_begin, k_end)
    sval, perm, rank, hs = l1.l1dm_debug_export(h)
    l1.l1dm_free(h)
    T, order = oracle.alg1(X[:, k_begin:k_end])
    assert np.array_equal(perm, order)
    assert np.array_equal(sval, T)          # -0.0 == +0.0 compares equal
    ar = np.arange(n, dtype=np.uint32)
    for k in range(k_end - k_begin):
        assert np.array_equal(rank[k][perm[k]], ar)
    href = X[:, k_begin:k_end].astype(np.float64).sum(1)
    assert np.allclose(hs, href, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("n,d", [(1, 1), (2, 3), (31, 2), (4095, 3), (4096, 2), (4097, 5),
                                 (12289, 4), (100003, 3)])
def test_sort_random_float(n, d):
    rng = np.random.default_rng(n * 31 + d)
    check_tables(rng.standard_normal((n, d)).astype(np.float32))


@pytest.mark.parametrize("n", [5000, 70001])
def test_sort_ties_and_special_values(n):
    rng = np.random.default_rng(n)
    X = rng.integers(-3, 4, size=(n, 6)).astype(np.float32)
    X[::5, 0] = -0.0
    X[1::5, 0] = 0.0
    X[:, 1] = np.float32(7.0)                                  # all equal (every pass trivial)
    X[::3, 2] = np.finfo(np.float32).max
    X[1::3, 2] = -np.finfo(np.float32).max
    X[::7, 3] = np.float32(1e-45)                              # denormals
    X[1::7, 3] = np.float32(-1e-45)
    X[:, 4] = rng.integers(0, 256, size=n).astype(np.float32)  # c5-like bytes
    check_tables(X)


def test_sort_all_passes_trivial_identity_path():
    X = np.full((3000, 4), 2.5, dtype=np.float32)
    check_tables(X)


def test_sort_shard_range():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((9000, 10)).astype(np.float32)
    check_tables(X, 3, 7)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_sort_workload_structure(name):
    w = wl.workload(name, n=50000, d=8)
    X = wl.make_points(w, "cuda").cpu().numpy()
    check_tables(X)


def test_nonfinite_rejected():
    X = np.ones((100, 3), dtype=np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        Xb = X.copy()
        Xb[57, 1] = bad
        with pytest.raises(l1.L1dmError) as e:
            l1.l1dm_prepare(torch.from_numpy(Xb).cuda())
        assert e.value.name == "L1DM_ENONFINITE"
