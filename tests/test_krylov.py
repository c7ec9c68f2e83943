"""Host logic of the matrix-free consumers with an injected CPU product:
A = the oracle's dense matrix (oracle.brute(X, I), pinned in test_oracle_pins.py), its
spectrum from numpy.linalg.eigh (a library routine).  The GPU runs are in test_gpu_krylov.py."""
import numpy as np
import pytest
import torch

import oracle
from paper_2210_15114_b200.krylov import block_krylov, cg_solve, lowrank_error


def dense_matvec(A):
    At = torch.from_numpy(A)
    return lambda V: At @ V.to(torch.float64)


def l1_matrix(n, d, seed):
    X = np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)
    return oracle.brute(X, np.eye(n, dtype=np.float32))


def test_topk_singular_values_match_dense_spectrum():
    A = l1_matrix(300, 5, 0)
    sv = np.sort(np.abs(np.linalg.eigvalsh(A)))[::-1]
    r = block_krylov(dense_matvec(A), 300, 10, eps=0.5, seed=3)
    assert np.all(np.diff(r.sigma.numpy()) <= 0)                     # nonincreasing
    assert np.allclose(r.sigma.numpy(), sv[:10], rtol=1e-6)
    ZtZ = (r.Z.T @ r.Z).numpy()
    assert np.abs(ZtZ - np.eye(10)).max() <= 1e-8                    # orthonormal columns


def test_lowrank_relative_error_bound():
    """||A (I - Z Z^T)||_F <= (1 + eps) ||A - A_k||_F (Thm. opt_lowrank_p)."""
    A = l1_matrix(300, 5, 1)
    lam = np.linalg.eigvalsh(A)
    k = 10
    best = np.sqrt(np.sort(lam ** 2)[:-k].sum())                     # ||A - A_k||_F
    r = block_krylov(dense_matvec(A), 300, k, eps=0.5, seed=4)
    Z = r.Z.numpy()
    err = np.linalg.norm(A - (A @ Z) @ Z.T)
    assert err <= 1.5 * best
    est = np.sqrt(lowrank_error(dense_matvec(A), r.Z, probes=64))
    assert 0.5 * err <= est <= 2 * err                                # Hutchinson estimate


def test_exact_rank_one_gram():
    """Points on a line through the origin, Gram kernel: rank 1, sigma_1 = ||x||^2 n-ish."""
    n = 120
    X = (np.arange(n)[:, None] * np.array([[1.0, 2.0]])).astype(np.float64)
    A = X @ X.T
    r = block_krylov(dense_matvec(A), n, 1, seed=5)
    assert abs(r.sigma[0].item() - np.linalg.norm(X) ** 2) <= 1e-8 * np.linalg.norm(X) ** 2
    Z = r.Z.numpy()
    assert np.linalg.norm(A - (A @ Z) @ Z.T) <= 1e-8 * np.linalg.norm(A)


def test_cg_spd_and_normal_equations():
    rng = np.random.default_rng(6)
    X = rng.standard_normal((200, 240))
    A = X @ X.T + 1e-1 * np.eye(200)                                  # SPD (Gram + ridge)
    b = torch.from_numpy(rng.standard_normal(200))
    res = cg_solve(dense_matvec(A), b, tol=1e-10, maxit=1000)
    assert res.converged and res.residual <= 1e-8
    L = l1_matrix(150, 4, 7)                                          # symmetric indefinite
    res2 = cg_solve(dense_matvec(L), torch.from_numpy(rng.standard_normal(150)), tol=1e-9,
                    maxit=5000, normal_equations=True)
    assert res2.residual <= 1e-6
    bad = cg_solve(dense_matvec(A), b, tol=1e-14, maxit=2)            # reported, not silent
    assert not bad.converged and bad.iterations == 2


def test_rejects_bad_k():
    with pytest.raises(ValueError):
        block_krylov(dense_matvec(np.eye(4)), 4, 4)
