"""Pins for the oracle's approximate-l2 pieces (Thm. l2embed P:623-631,
Thm. l2_approx): the embedding against an exact library matmul on integer data, its
zero/linearity, the constant beta = sqrt(2/pi), the exact l2 product against hand
values and the Pythagorean 3-4-5 case, and the theorem's (1 +- eps) guarantee statistically."""
import math

import numpy as np
import pytest

import oracle
from paper_2210_15114_b200.l2approx import embedding_dim

RNG = np.random.default_rng(2022)
BETA = 0.7978845608028654   # sqrt(2/pi), "0.7978845608..."


def test_embed_matches_exact_matmul_and_is_linear():
    X = RNG.integers(-3, 4, size=(20, 5))
    G = RNG.integers(-2, 3, size=(9, 5))
    want = ((X @ G.T) / (BETA * 9)).astype(np.float32)          # int64 matmul, then one rounding
    got = oracle.l2_embed(X.astype(np.float32), G.astype(np.float32))
    assert np.array_equal(got, want)
    assert np.all(oracle.l2_embed(np.zeros((3, 5), np.float32), G.astype(np.float32)) == 0)
    assert abs(math.sqrt(2 / math.pi) - BETA) < 1e-15


def test_exact_l2_product_hand_values():
    """x1 = (0,0), x2 = (3,4), x3 = (0,4): D12 = 5, D13 = 4, D23 = 3; z = (1,1,1) -> (9,8,7)."""
    X = np.array([[0, 0], [3, 4], [0, 4]], dtype=np.float32)
    assert np.array_equal(oracle.brute_l2(X, np.ones((3, 1), np.float32))[:, 0], [9.0, 8.0, 7.0])
    assert np.all(oracle.brute_l2(np.tile(X[:1], (4, 1)), np.ones((4, 2), np.float32)) == 0)


def test_embedding_preserves_norms_statistically():
    """Thm. l2embed: ||T x||_1 in [(1-eps), (1+eps)] ||x||_2 for >= 95% of unit vectors at
    k = ceil(12 ln n / eps^2) (200 random unit vectors, eps = 0.2)."""
    eps, d = 0.2, 30
    k = embedding_dim(200, eps)
    G = RNG.standard_normal((k, d)).astype(np.float32)
    U = RNG.standard_normal((200, d))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    norms = np.abs(oracle.l2_embed(U.astype(np.float32), G).astype(np.float64)).sum(1)
    assert np.mean(np.abs(norms - 1.0) <= eps) >= 0.95


def test_l1_of_embedding_approximates_l2_matrix():
    """Thm. l2_approx: B_ij = ||x'_i - x'_j||_1 within 1 +- 1.25 eps of ||x_i - x_j||_2 for
    >= 95% of entries (n = 100, eps = 0.2); and ||A - B||_F <= eps ||A||_F."""
    eps, n, d = 0.2, 100, 8
    X = RNG.standard_normal((n, d)).astype(np.float32)
    G = RNG.standard_normal((embedding_dim(n, eps), d)).astype(np.float32)
    Xp = oracle.l2_embed(X, G)
    I = np.eye(n, dtype=np.float32)
    A = oracle.brute_l2(X, I)
    B = oracle.brute(Xp, I)
    off = ~np.eye(n, dtype=bool)
    ratio = B[off] / A[off]
    assert np.mean(np.abs(ratio - 1) <= 1.25 * eps) >= 0.95
    assert np.linalg.norm(A - B) <= eps * np.linalg.norm(A)
