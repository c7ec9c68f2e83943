"""Pins for the CPU oracle (oracle/), each against something other than the oracle itself.

Pin ids follow SURVEY.md §8(c) / DESIGN.md §3.  These run without a GPU.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, col_rel_l2, load_golden

RNG = np.random.default_rng(20221027)


def rand_instance(rng, n, d, m, integer):
    if integer:
        X = rng.integers(0, 4, size=(n, d)).astype(np.float32)
    else:
        X = rng.standard_normal((n, d)).astype(np.float32)
    Z = rng.standard_normal((n, m)).astype(np.float32)
    return X, Z


# ---- Q1, Q2, Q20, Q21: hand-derived golden fixtures --------------------------------------
@pytest.mark.parametrize("name", GOLDEN)
def test_golden_all_modes(name):
    X, Z, Y = load_golden(name)
    assert np.array_equal(oracle.brute(X, Z), Y)
    assert np.array_equal(oracle.sort_based(X, Z), Y)
    assert np.array_equal(oracle.rows(X, Z, np.arange(X.shape[0])), Y)
    if np.all(X >= 0):
        assert np.array_equal(oracle.hist(X, Z, M=int(X.max())), Y.astype(np.int64))


# ---- Q3: degenerate inputs --------------------------------------------------------------
def test_zero_query_and_equal_points_and_single_point():
    X, Z = rand_instance(RNG, 17, 3, 4, False)
    assert np.all(oracle.brute(X, np.zeros_like(Z)) == 0)
    assert np.all(oracle.sort_based(X, np.zeros_like(Z)) == 0)
    Xe = np.tile(X[:1], (17, 1))
    assert np.all(oracle.brute(Xe, Z) == 0)
    assert np.all(oracle.sort_based(Xe, Z) == 0)
    assert np.all(oracle.sort_based(X[:1], Z[:1]) == 0)
    assert np.all(oracle.brute(X[:1], Z[:1]) == 0)


# ---- Q4: zero diagonal, (A e_j)_j = 0 ----------------------------------------------------
def test_zero_diagonal():
    X, _ = rand_instance(RNG, 40, 5, 1, False)
    E = np.eye(40, dtype=np.float32)
    A_b = oracle.brute(X, E)
    A_s = oracle.sort_based(X, E)
    assert np.all(np.diag(A_b) == 0)
    assert np.all(np.abs(np.diag(A_s)) <= 1e-12 * np.abs(A_s).max())
    # A itself against pairwise distances from numpy (a library evaluation of P:149)
    D = np.abs(X[:, None, :].astype(np.float64) - X[None, :, :].astype(np.float64)).sum(-1)
    assert np.allclose(A_b, D, rtol=1e-14, atol=0)
    assert np.allclose(A_s, D, rtol=1e-12, atol=1e-12)


# ---- Q5, Q6: symmetry via queries, linearity ---------------------------------------------
def test_symmetry_and_linearity():
    X, Z = rand_instance(RNG, 64, 6, 3, False)
    z, w = Z[:, 0], Z[:, 1]
    for f in (oracle.brute, oracle.sort_based):
        lhs = float(np.dot(z.astype(np.float64), f(X, w)))
        rhs = float(np.dot(w.astype(np.float64), f(X, z)))
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)
    a = np.float32(0.5)  # exact in fp32, so z + a*w is computed exactly here for small ints
    Xi, Zi = rand_instance(RNG, 64, 6, 2, True)
    Zi = np.round(Zi * 4).astype(np.float32)
    z1, z2 = Zi[:, 0], Zi[:, 1]
    comb = (z1 + a * z2).astype(np.float32)
    for f in (oracle.brute, oracle.sort_based):
        assert np.array_equal(f(Xi, comb), f(Xi, z1) + 0.5 * f(Xi, z2))


# ---- Q7: collinear equally spaced points, closed form -------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 10, 37])
def test_collinear_closed_form(n):
    u = np.array([1, -2, 0, 3], dtype=np.float32)
    X = (np.arange(n, dtype=np.float32)[:, None] * u[None, :]).astype(np.float32)
    one = np.ones(n, dtype=np.float32)
    norm_u = float(np.abs(u).sum())
    i = np.arange(n)
    expect = norm_u * (i * (i + 1) / 2 + (n - 1 - i) * (n - i) / 2)
    for f in (oracle.brute, oracle.sort_based):
        y = f(X, one)
        assert np.array_equal(y, expect)
        assert y.sum() == norm_u * (n ** 3 - n) / 3


# ---- Q8: 1^T A 1 = 2 sum_k sum_{i<j} |x_ik - x_jk| via sorted values, exact rationals --------
def test_total_sum_closed_form():
    X, _ = rand_instance(RNG, 50, 4, 1, False)
    n, d = X.shape
    total = Fraction(0)
    for k in range(d):
        v = np.sort(X[:, k])
        for r in range(n):
            total += (2 * r - n + 1) * Fraction(float(v[r]))
    total *= 2
    one = np.ones(n, dtype=np.float32)
    for f in (oracle.brute, oracle.sort_based):
        s = float(np.sum(f(X, one), dtype=np.float64))
        assert abs(s - float(total)) <= 1e-12 * abs(float(total))


# ---- Q9: Hamming special case, A Z = h(1^T Z) + 1(h^T Z) - 2 X (X^T Z) (library matmul) -----
def test_hamming_identity():
    rng = np.random.default_rng(9)
    X = rng.integers(0, 2, size=(80, 11)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(80, 5)).astype(np.float32)
    Xi, Zi = X.astype(np.int64), Z.astype(np.int64)
    h = Xi.sum(1)
    expect = np.outer(h, Zi.sum(0)) + np.outer(np.ones(80, np.int64), h @ Zi) - 2 * Xi @ (Xi.T @ Zi)
    assert np.array_equal(oracle.brute(X, Z), expect.astype(np.float64))
    assert np.array_equal(oracle.sort_based(X, Z), expect.astype(np.float64))
    assert np.array_equal(oracle.hist(X, Z, M=1), expect)


# ---- Q10: exact integer path (HIST) equals brute force exactly ------------------------------
def test_hist_exact_against_brute():
    rng = np.random.default_rng(10)
    X = rng.integers(0, 256, size=(300, 9)).astype(np.float32)
    Z = (2 * rng.integers(0, 2, size=(300, 4)) - 1).astype(np.float32)
    Yh = oracle.hist(X, Z, M=255)
    assert np.array_equal(oracle.brute(X, Z), Yh.astype(np.float64))
    assert np.array_equal(oracle.sort_based(X, Z), Yh.astype(np.float64))
    with pytest.raises(ValueError):
        oracle.hist(X + 0.5, Z, M=255)


# ---- Q11: Alg.1+Alg.2 against brute force on 1000 random small instances -----------------
def test_sort_based_vs_brute_many():
    rng = np.random.default_rng(11)
    worst = 0.0
    for t in range(1000):
        n = int(rng.integers(1, 65))
        d = int(rng.integers(1, 9))
        m = int(rng.integers(1, 9))
        X, Z = rand_instance(rng, n, d, m, integer=(t % 2 == 0))
        Yb = oracle.brute(X, Z, nthreads=1)
        Ys = oracle.sort_based(X, Z, nthreads=1)
        if t % 2 == 0:
            assert np.array_equal(Yb, Ys)
        worst = max(worst, col_rel_l2(Ys, Yb) if np.any(Yb) else 0.0)
    assert worst <= 1e-12


# ---- Q13: Alg. 1 tables against numpy's stable argsort (library routine) ------------------
def test_alg1_matches_stable_argsort():
    rng = np.random.default_rng(13)
    X = rng.integers(-3, 4, size=(500, 6)).astype(np.float32)
    X[::7, 2] = -0.0
    X[:, 5] = rng.standard_normal(500).astype(np.float32)
    T, order = oracle.alg1(X)
    for k in range(X.shape[1]):
        ref = np.argsort(X[:, k], kind="stable")
        assert np.array_equal(order[k], ref.astype(np.uint32))
        assert np.array_equal(T[k], X[ref, k])
        assert np.all(np.diff(T[k]) >= 0)
    Xbad = X.copy()
    Xbad[3, 1] = np.nan
    with pytest.raises(ValueError):
        oracle.alg1(Xbad)


# ---- Q14: invariances (exact on integer data) ------------------------------------------
def test_invariances_integer_data():
    rng = np.random.default_rng(14)
    X = rng.integers(0, 6, size=(70, 5)).astype(np.float32)
    Z = rng.integers(-4, 5, size=(70, 3)).astype(np.float32)
    Y = oracle.brute(X, Z)
    Ys = oracle.sort_based(X, Z)
    assert np.array_equal(Y, Ys)
    shift = np.array([3, -7, 100, 0, -1], dtype=np.float32)
    assert np.array_equal(oracle.sort_based(X + shift, Z), Y)        # translation
    assert np.array_equal(oracle.sort_based(-X, Z), Y)               # reflection
    p = rng.permutation(70)
    assert np.array_equal(oracle.sort_based(X[p], Z[p]), Y[p])       # permute points
    q = rng.permutation(5)
    assert np.array_equal(oracle.sort_based(X[:, q], Z), Y)          # permute coordinates


# ---- Q15 (oracle level): coordinate additivity of the partial products ---------------
def test_coordinate_shards_sum_to_whole():
    rng = np.random.default_rng(15)
    X = rng.integers(0, 9, size=(90, 7)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(90, 3)).astype(np.float32)
    _, order = oracle.alg1(X)
    whole = oracle.alg2(X, order, Z)
    parts = [oracle.alg2_range(X, order, a, b, Z) for a, b in [(0, 2), (2, 3), (3, 7)]]
    assert np.array_equal(sum(parts), whole)
    assert np.array_equal(parts[0], oracle.brute(X[:, 0:2], Z))


# ---- Q16: nonnegativity, Q17: n = 2 -----------------------------------------------------
def test_sign_and_two_points():
    rng = np.random.default_rng(16)
    X, _ = rand_instance(rng, 30, 4, 1, False)
    z = np.abs(rng.standard_normal(30)).astype(np.float32)
    assert np.all(oracle.brute(X, z) >= 0)
    assert np.all(oracle.sort_based(X, z) >= -1e-12)
    X2 = np.array([[1.5, -2.0, 0.25], [-0.5, 1.0, 0.25]], dtype=np.float32)
    D = 2.0 + 3.0 + 0.0
    Z2 = np.array([[2.0, 1.0], [-3.0, 5.0]], dtype=np.float32)
    expect = np.array([[D * -3.0, D * 5.0], [D * 2.0, D * 1.0]])
    assert np.array_equal(oracle.brute(X2, Z2), expect)
    assert np.array_equal(oracle.sort_based(X2, Z2), expect)


# ---- rows(): the definition for selected rows equals the full evaluation ---------------------
def test_rows_subset_matches_full():
    X, Z = rand_instance(RNG, 120, 5, 3, False)
    r = np.array([0, 119, 7, 7, 64])
    assert np.array_equal(oracle.rows(X, Z, r), oracle.brute(X, Z)[r])


# ---- thread-count independence ----------------------------------------------------------
def test_thread_count_independent():
    X, Z = rand_instance(RNG, 200, 6, 5, False)
    a = oracle.sort_based(X, Z, nthreads=1)
    b = oracle.sort_based(X, Z, nthreads=3)
    assert np.array_equal(a, b)
    assert np.array_equal(oracle.brute(X, Z, nthreads=1), oracle.brute(X, Z, nthreads=4))


# ---- Q18: precision discriminator for the U-form (DESIGN.md §3 tolerance derivation) -------
def test_u_form_precision_requires_fp64_storage():
    """The U-form evaluated with numpy in fp64 meets the 1e-9 bar against the
    oracle; the same with U rounded to fp32 before the point gather does not, which
    is why the library keeps U (and every accumulator) in fp64."""
    rng = np.random.default_rng(18)
    n, d = 1 << 15, 4
    centres = rng.uniform(-10, 10, size=(32, d))
    X = (centres[rng.integers(0, 32, n)] + 0.5 * rng.standard_normal((n, d))).astype(np.float32)
    z = rng.standard_normal(n).astype(np.float32)
    rows = np.arange(0, n, 997)
    ref = oracle.rows(X, z[:, None], rows)[:, 0]

    def u_form(store):
        y = np.zeros(n)
        S = z.astype(np.float64).sum()
        for k in range(d):
            order = np.argsort(X[:, k], kind="stable")
            v = X[order, k].astype(np.float64)
            s = z[order].astype(np.float64)
            P = np.concatenate([[0.0], np.cumsum(s)[:-1]])
            Q = np.concatenate([[0.0], np.cumsum(v * s)[:-1]])
            U = store(v * P - Q)
            T = (v * s).sum()
            contrib = np.empty(n)
            contrib[order] = 2 * U + T - v * S
            y += contrib
        return y[rows]

    err64 = np.linalg.norm(u_form(lambda u: u) - ref) / np.linalg.norm(ref)
    err32 = np.linalg.norm(u_form(lambda u: u.astype(np.float32).astype(np.float64)) - ref) / \
        np.linalg.norm(ref)
    assert err64 <= 1e-12
    assert err32 > 1e-9


# ---- Q19: the U-form scan identity the CUDA path evaluates ------
def test_u_form_scan_identity_against_direct_sums():
    """Per coordinate: U_r = sum_{j: rho(j) < r} z_j (v_r - x_jk) written as a direct O(n^2) sum
    equals v_r P_r - Q_r from exclusive prefixes, and sum_j z_j |x_ik - x_jk| equals
    2 U_rho(i) + T - x_ik S for every point — with ties (integer coordinates), where either side
    of a tie may hold the equal values.  Exact in rationals on integer data."""
    rng = np.random.default_rng(19)
    for trial in range(40):
        n = int(rng.integers(1, 40))
        x = rng.integers(-4, 5, size=n).astype(np.int64)
        z = rng.integers(-3, 4, size=n).astype(np.int64)
        order = np.argsort(x, kind="stable")
        rho = np.empty(n, dtype=np.int64)
        rho[order] = np.arange(n)
        v, s = x[order], z[order]
        P = np.concatenate([[0], np.cumsum(s)[:-1]])
        Q = np.concatenate([[0], np.cumsum(v * s)[:-1]])
        U = v * P - Q
        U_direct = np.array([sum(z[j] * (v[r] - x[j]) for j in range(n) if rho[j] < r)
                             for r in range(n)], dtype=np.int64)
        assert np.array_equal(U, U_direct)
        S, T = z.sum(), (x * z).sum()
        lhs = np.array([sum(z[j] * abs(x[i] - x[j]) for j in range(n)) for i in range(n)])
        assert np.array_equal(lhs, 2 * U[rho] + T - x * S)
