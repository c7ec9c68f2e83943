"""Sort-free even-p l_p^p (p = 2 squared Euclidean, 4, 6) through the C ABI
against the oracle.  Tolerance 1e-9 (per-column relative l2; fp64 moments of fp32 inputs, the
same bar as l1; R18); integer data with small moments bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_15114_b200 as l1
from conftest import GOLDEN_EVEN, col_rel_l2, golden_p, load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", GOLDEN_EVEN)
def test_even_goldens_exact(name):
    X, Z, Y = load_golden(name)
    Yg = l1.l1dm_lpp_even_matvec(torch.from_numpy(X).cuda(), golden_p(name),
                                 torch.from_numpy(Z).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(Yg.cpu().numpy(), Y)


# tiles of 64 points / 64 coordinates / 64 columns, ragged in every dimension
@pytest.mark.parametrize("p", [2, 4, 6])
@pytest.mark.parametrize("n,d,m", [(1, 1, 1), (5, 3, 2), (65, 63, 65), (1000, 7, 3),
                                   (3001, 130, 17), (20000, 16, 64),
                                   (3001, 128, 20), (1500, 256, 68)])  # cp.async ring K12
def test_even_random_vs_oracle(n, d, m, p):
    rng = np.random.default_rng(n + 10 * d + 100 * m + p)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Z = rng.standard_normal((n, m)).astype(np.float32)
    Yg = l1.l1dm_lpp_even_matvec(torch.from_numpy(X).cuda(), p, torch.from_numpy(Z).cuda())
    torch.cuda.synchronize()
    # natural scale of a column (moment terms cancel to the result): sum_k (2 max|x_k|)^p ||z||
    floor = float(((2 * np.abs(X).max(0).astype(np.float64)) ** p).sum() * np.linalg.norm(Z, axis=0).max())
    if n <= 3001:
        Yr = oracle.brute_lp(X, Z, p)
        assert col_rel_l2(Yg.cpu().numpy(), Yr, floor=1e-3 * floor) <= 1e-9
    else:
        rows = np.array([0, 1, 777, n - 1])
        Yr = oracle.rows_lp(X, Z, p, rows)
        assert col_rel_l2(Yg[torch.from_numpy(rows).cuda()].cpu().numpy(), Yr) <= 1e-9


def test_even_integer_exact_and_host_strided():
    rng = np.random.default_rng(3)
    X = rng.integers(-4, 5, size=(2000, 9)).astype(np.float32)
    Zw = rng.integers(-2, 3, size=(2000, 7)).astype(np.float32)
    Z = Zw[:, 1:5]                                           # strided host view
    Y = l1.l1dm_lpp_even_matvec(X, 2, Z)                     # host in, host out
    assert np.array_equal(Y.numpy(), oracle.lp_even(X, np.ascontiguousarray(Z), 2))
    Y4 = l1.l1dm_lpp_even_matvec(torch.from_numpy(X).cuda(), 4, torch.from_numpy(Zw).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(Y4.cpu().numpy(), oracle.lp_even(X, Zw, 4))


def test_even_rejects_bad_p():
    X = torch.zeros((10, 2), device="cuda")
    Z = torch.zeros((10, 1), device="cuda")
    for bad in (0, 1, 3, 8):
        with pytest.raises(l1.L1dmError):
            l1.l1dm_lpp_even_matvec(X, bad, Z)


# ---- Thm. maha's bilinear form ----------------------------------------------------------
def test_bilinear_golden_and_identity():
    X = np.array([[1, 0], [0, 2]], dtype=np.float32)
    M = np.array([[1, 2], [3, 4]], dtype=np.float64)
    Y = l1.l1dm_bilinear_matvec(torch.from_numpy(X).cuda(), torch.from_numpy(M).cuda(),
                                torch.ones((2, 1), device="cuda"))
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy()[:, 0], [5.0, 22.0])
    rng = np.random.default_rng(4)
    Xi = rng.integers(-4, 5, size=(3000, 70)).astype(np.float32)
    Zi = rng.integers(-3, 4, size=(3000, 9)).astype(np.float32)
    Mi = rng.integers(-2, 3, size=(70, 70)).astype(np.float64)
    Yg = l1.l1dm_bilinear_matvec(Xi, Mi, Zi)              # host in, host out: exact integers
    assert np.array_equal(Yg.numpy(), oracle.brute_bilinear(Xi, Mi, Zi))


@pytest.mark.parametrize("n,d,m", [(1, 1, 1), (65, 63, 65), (2000, 130, 17)])
def test_bilinear_random_vs_oracle(n, d, m):
    rng = np.random.default_rng(n + d + m)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Z = rng.standard_normal((n, m)).astype(np.float32)
    M = rng.standard_normal((d, d))
    Yg = l1.l1dm_bilinear_matvec(torch.from_numpy(X).cuda(), torch.from_numpy(M).cuda(),
                                 torch.from_numpy(Z).cuda())
    torch.cuda.synchronize()
    Yr = oracle.brute_bilinear(X, M, Z)
    scale = float(np.abs(X).sum(1).max() ** 2 * np.abs(M).max() * np.abs(Z).sum(0).max())
    assert col_rel_l2(Yg.cpu().numpy(), Yr, floor=1e-6 * scale) <= 1e-9


def test_handleless_launch_counter():
    """The handle-free entries count their kernels (bench.py's gpu_launches for even p)."""
    X = torch.randn(300, 9, device="cuda")
    Z = torch.randn(300, 4, device="cuda")
    c0 = l1.l1dm_handleless_launches()
    l1.l1dm_lpp_even_matvec(X, 2, Z)
    c1 = l1.l1dm_handleless_launches()
    l1.l1dm_bilinear_matvec(X, torch.eye(9, dtype=torch.float64, device="cuda"), Z)
    c2 = l1.l1dm_handleless_launches()
    l1.l1dm_l2_embed(X, torch.randn(16, 9, device="cuda"))
    c3 = l1.l1dm_handleless_launches()
    torch.cuda.synchronize()
    assert (c1 - c0, c2 - c1, c3 - c2) == (4, 5, 1)
