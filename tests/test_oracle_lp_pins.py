"""Pins for the oracle's l_p^p (odd p) and TV functions, each against
something other than the oracle itself: hand-derived goldens, the pinned l1 oracle on data
where |a-b|^p = |a-b|, exact closed forms, exact symmetries.  No GPU needed.

  brute_lp   the definition  sum_j z_j sum_k |x_ik - x_jk|^p          (Thm. odd_p)
  lp_sorted  SPEC S:150-158's sort-based construction in Alg. 2's shape (odd p)
  brute_tv   TV(x, y) = ||x - y||_1 / 2                               (Thm. tv)
"""
import numpy as np
import pytest

import oracle
from conftest import GOLDEN_LP, GOLDEN_TV, golden_p, load_golden

RNG = np.random.default_rng(31)
ODD = [1, 3, 5, 7]


@pytest.mark.parametrize("name", GOLDEN_LP)
def test_lp_goldens(name):
    X, Z, Y = load_golden(name)
    p = golden_p(name)
    assert np.array_equal(oracle.brute_lp(X, Z, p), Y)
    assert np.array_equal(oracle.lp_sorted(X, Z, p), Y)


@pytest.mark.parametrize("name", GOLDEN_TV)
def test_tv_golden(name):
    X, Z, Y = load_golden(name)
    assert np.array_equal(oracle.brute_tv(X, Z), Y)


@pytest.mark.parametrize("p", ODD)
def test_p1_is_l1_and_binary_data_is_l1_for_every_p(p):
    """|a - b|^p = |a - b| when |a - b| in {0, 1}: A_p = A_1 exactly (A_1 pinned by Q1-Q21)."""
    X = RNG.integers(0, 2, size=(37, 6)).astype(np.float32)
    Z = RNG.integers(-3, 4, size=(37, 3)).astype(np.float32)
    Y1 = oracle.brute(X, Z)
    assert np.array_equal(oracle.brute_lp(X, Z, p), Y1)
    assert np.array_equal(oracle.lp_sorted(X, Z, p), Y1)
    Xf = RNG.standard_normal((23, 3)).astype(np.float32)
    Zf = RNG.standard_normal((23, 2)).astype(np.float32)
    assert np.array_equal(oracle.brute_lp(Xf, Zf, 1), oracle.brute(Xf, Zf))


@pytest.mark.parametrize("p", [3, 5, 7])
def test_collinear_closed_form(p):
    """x_i = i u (u integer): (A_p 1)_i = ||u||_p^p (sum_{a=1}^{i} a^p + sum_{a=1}^{n-1-i} a^p),
    evaluated in exact Python integers."""
    n = 21
    u = np.array([1, -2, 3], dtype=np.int64)
    X = (np.arange(n)[:, None] * u[None, :]).astype(np.float32)
    up = int(sum(abs(int(v)) ** p for v in u))
    want = np.array([up * (sum(a ** p for a in range(1, i + 1)) +
                           sum(a ** p for a in range(1, n - i))) for i in range(n)],
                    dtype=np.float64)
    ones = np.ones((n, 1), dtype=np.float32)
    assert np.array_equal(oracle.brute_lp(X, ones, p)[:, 0], want)
    assert np.array_equal(oracle.lp_sorted(X, ones, p)[:, 0], want)


@pytest.mark.parametrize("p", [3, 5])
def test_exact_symmetries_on_integer_data(p):
    """A_p depends on |x_ik - x_jk| only: integer shifts and reflection leave it unchanged;
    scaling by 2 multiplies it by 2^p; permuting points permutes Y's rows (all exact)."""
    X = RNG.integers(-4, 5, size=(30, 4)).astype(np.float32)
    Z = RNG.integers(-2, 3, size=(30, 2)).astype(np.float32)
    Y = oracle.brute_lp(X, Z, p)
    assert np.array_equal(oracle.lp_sorted(X, Z, p), Y)
    assert np.array_equal(oracle.lp_sorted(X + 7, Z, p), Y)
    assert np.array_equal(oracle.lp_sorted(-X, Z, p), Y)
    assert np.array_equal(oracle.lp_sorted(2 * X, Z, p), (2.0 ** p) * Y)
    perm = RNG.permutation(30)
    assert np.array_equal(oracle.lp_sorted(X[perm], Z[perm], p), Y[perm])


@pytest.mark.parametrize("p", [3, 5, 7])
def test_sorted_route_matches_definition(p):
    """Two independent routes (sort + moments vs pairwise powers), random float instances and
    tie-heavy integer instances; plus z^T A w = w^T A z."""
    for trial in range(40):
        n, d, m = int(RNG.integers(1, 40)), int(RNG.integers(1, 6)), int(RNG.integers(1, 4))
        if trial % 2:
            X = RNG.integers(0, 4, size=(n, d)).astype(np.float32)
            Z = RNG.integers(-3, 4, size=(n, m)).astype(np.float32)
            assert np.array_equal(oracle.lp_sorted(X, Z, p), oracle.brute_lp(X, Z, p))
        else:
            X = RNG.standard_normal((n, d)).astype(np.float32)
            Z = RNG.standard_normal((n, m)).astype(np.float32)
            a, b = oracle.lp_sorted(X, Z, p), oracle.brute_lp(X, Z, p)
            assert np.abs(a - b).max() <= 1e-12 * max(np.abs(b).max(), 1e-300)
    X = RNG.standard_normal((50, 3)).astype(np.float32)
    zw = RNG.standard_normal((50, 2)).astype(np.float32)
    Y = oracle.brute_lp(X, zw, p)
    lhs, rhs = float(zw[:, 0] @ Y[:, 1]), float(zw[:, 1] @ Y[:, 0])
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_rows_lp_equals_brute_rows():
    X = RNG.standard_normal((60, 4)).astype(np.float32)
    Z = RNG.standard_normal((60, 2)).astype(np.float32)
    rows = np.array([0, 7, 59, 7])
    for p in (1, 3, 5):
        assert np.array_equal(oracle.rows_lp(X, Z, p, rows), oracle.brute_lp(X, Z, p)[rows])


def test_tv_is_half_l1_on_simplex_rows():
    X = RNG.dirichlet(np.ones(5), size=40).astype(np.float32)
    Z = RNG.standard_normal((40, 3)).astype(np.float32)
    assert np.array_equal(oracle.brute_tv(X, Z), 0.5 * oracle.brute(X, Z))   # power-of-2 scale
    E = np.eye(40, dtype=np.float32)[:, :2]                                   # z = e_1: TV column
    col = oracle.brute_tv(X, E)[:, 0]
    assert np.all(col >= 0) and np.all(col <= 1 + 1e-6) and col[0] == 0


def test_lp_rejects_even_p_in_sorted_route():
    X = np.zeros((3, 1), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle.lp_sorted(X, np.ones((3, 1), dtype=np.float32), 2)


# ---- even p (NEXT-4): brute_lp (definition) and lp_even (Alg. query_p_even, corrected) ----
from conftest import GOLDEN_EVEN  # noqa: E402


@pytest.mark.parametrize("name", GOLDEN_EVEN)
def test_even_goldens(name):
    X, Z, Y = load_golden(name)
    p = golden_p(name)
    assert np.array_equal(oracle.brute_lp(X, Z, p), Y)
    assert np.array_equal(oracle.lp_even(X, Z, p), Y)


def test_l2sq_gram_identity_exact():
    """||a - b||^2 = ||a||^2 + ||b||^2 - 2 a.b: A_2 Z = h (1^T Z) + 1 (h^T Z) - 2 X (X^T Z),
    evaluated with numpy int64 matmul on integer data (a library routine, exact)."""
    X = RNG.integers(-5, 6, size=(40, 7))
    Z = RNG.integers(-3, 4, size=(40, 3))
    h = (X * X).sum(1)
    want = h[:, None] * Z.sum(0)[None, :] + (h @ Z)[None, :] - 2 * (X @ (X.T @ Z))
    Xf, Zf = X.astype(np.float32), Z.astype(np.float32)
    assert np.array_equal(oracle.brute_lp(Xf, Zf, 2), want.astype(np.float64))
    assert np.array_equal(oracle.lp_even(Xf, Zf, 2), want.astype(np.float64))


@pytest.mark.parametrize("p", [2, 4, 6])
def test_even_routes_agree_and_collinear(p):
    n = 17
    u = np.array([2, -1], dtype=np.int64)
    X = (np.arange(n)[:, None] * u[None, :]).astype(np.float32)
    up = int(sum(abs(int(v)) ** p for v in u))
    want = np.array([up * (sum(a ** p for a in range(1, i + 1)) + sum(a ** p for a in range(1, n - i)))
                     for i in range(n)], dtype=np.float64)
    ones = np.ones((n, 1), dtype=np.float32)
    assert np.array_equal(oracle.brute_lp(X, ones, p)[:, 0], want)
    assert np.array_equal(oracle.lp_even(X, ones, p)[:, 0], want)
    Xf = RNG.standard_normal((30, 4)).astype(np.float32)
    Zf = RNG.standard_normal((30, 2)).astype(np.float32)
    a, b = oracle.lp_even(Xf, Zf, p), oracle.brute_lp(Xf, Zf, p)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


# ---- Thm. maha's bilinear form x^T M y (NEXT-4) -----------------------------------------
def test_bilinear_golden_hand_derived():
    """x1 = (1,0), x2 = (0,2), M = [[1,2],[3,4]] (not symmetric), z = (1,1):
    A11 = M00 = 1, A12 = 2 M01 = 4, A21 = 2 M10 = 6, A22 = 4 M11 = 16 -> y = (5, 22)."""
    X = np.array([[1, 0], [0, 2]], dtype=np.float32)
    M = np.array([[1, 2], [3, 4]], dtype=np.float64)
    Z = np.ones((2, 1), dtype=np.float32)
    assert np.array_equal(oracle.brute_bilinear(X, M, Z)[:, 0], [5.0, 22.0])
    assert np.array_equal(oracle.bilinear_alg(X, M, Z)[:, 0], [5.0, 22.0])


def test_bilinear_identity_is_gram_and_zero_and_routes_agree():
    X = RNG.integers(-4, 5, size=(30, 5))
    Z = RNG.integers(-3, 4, size=(30, 2))
    want = (X @ (X.T @ Z)).astype(np.float64)          # M = I: the Gram matvec
    Xf, Zf = X.astype(np.float32), Z.astype(np.float32)
    assert np.array_equal(oracle.brute_bilinear(Xf, np.eye(5), Zf), want)
    assert np.array_equal(oracle.bilinear_alg(Xf, np.eye(5), Zf), want)
    assert np.all(oracle.brute_bilinear(Xf, np.zeros((5, 5)), Zf) == 0)
    Mi = RNG.integers(-2, 3, size=(5, 5))              # integer M: X M X^T Z exactly (int64)
    assert np.array_equal(oracle.brute_bilinear(Xf, Mi.astype(np.float64), Zf),
                          (X @ Mi @ (X.T @ Z)).astype(np.float64))
    Mf = RNG.standard_normal((5, 5))
    Xr = RNG.standard_normal((30, 5)).astype(np.float32)
    a, b = oracle.bilinear_alg(Xr, Mf, Zf), oracle.brute_bilinear(Xr, Mf, Zf)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
