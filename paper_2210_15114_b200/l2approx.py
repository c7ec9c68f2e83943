"""Approximate l2 distance-matrix products through the l1 engine (
Thm. l2embed, Alg. "Preprocessing" for l2 and Thm. l2_approx).

    X' = X G^T / (beta k),  G: k x d i.i.d. N(0,1),  beta = sqrt(2/pi)     (l1dm_l2_embed)
    then the l1 product on X':  B Z with B_ij = ||x'_i - x'_j||_1 = (1 +- eps) ||x_i - x_j||_2

k = ceil(alpha log(n) / eps^2) (Thm. l2embed's O(log n / eps^2); alpha = 12 by default, the
SPEC's S:244 constant).  Composition of library calls only (the embedding GEMM and every query
run in libl1dm.so); G comes from the seeded generators in workloads.py.
"""
from __future__ import annotations

import math

import torch

from . import binding
from .workloads import gaussian_embedding


def embedding_dim(n: int, eps: float, alpha: float = 12.0) -> int:
    if not (0.0 < eps < 1.0):
        raise ValueError("0 < eps < 1")
    return max(1, math.ceil(alpha * math.log(max(n, 2)) / (eps * eps)))


class L2Approx:
    """Prepared approximate-l2 engine: X' = T X then the l1 prepare (Alg. 1) on X'."""

    def __init__(self, X: torch.Tensor, eps: float = 0.2, seed: int = 0, k: int | None = None,
                 alpha: float = 12.0):
        n, d = X.shape
        self.k = k or embedding_dim(n, eps, alpha)
        self.G = gaussian_embedding(self.k, d, seed, X.device)
        self.Xp = binding.l1dm_l2_embed(X, self.G)
        self.handle = binding.l1dm_prepare(self.Xp)

    def matvec(self, Z: torch.Tensor, Y: torch.Tensor | None = None) -> torch.Tensor:
        return binding.l1dm_matvec(self.handle, Z, Y)

    def close(self):
        binding.l1dm_free(self.handle)
        self.handle = None
