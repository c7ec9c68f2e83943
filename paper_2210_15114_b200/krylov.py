"""Matrix-free consumers of the block product (PAPER.md §"Applications",
P:727-817): randomized block Krylov for the top-k singular values / a rank-k approximation
(Thm. musco P:735-739 and Thm. bakshi22 P:727-731 as used by Thm. opt_lowrank_p, P:757-766;
SPEC S:340-357) and conjugate gradients (Thm. linear_system).

Every step runs in libl1dm.so (include/l1dm.h "Matrix-free consumers"): the products, the fp64
tensor-core GEMMs of the block Gram-Schmidt, CholeskyQR2 inside each block, the top-k
eigensolver of the Rayleigh quotient (Householder tridiagonalisation, bisection, inverse
iteration), and CG's dot products and updates with device scalars.  This module only
chooses the parameters, draws the start block (the method's random numbers, an input to the
library) and marshals results.  There is no host or torch fallback: without the library and a
B200 the calls raise.

Block Krylov (Musco & Musco's block Krylov iteration for symmetric A, whose singular values
are |eigenvalues|):
  K = [A Pi, A^2 Pi, ..., A^q Pi]  built block by block, each new block orthonormalised
  against the previous ones (block Gram-Schmidt: the last two blocks, then the whole basis) and
  within itself (CholeskyQR2); Rayleigh-Ritz: T = Q^T (A Q) from the orthogonalisation
  coefficients (block Lanczos with full re-orthogonalisation), its k eigenpairs of largest
  |lambda|, sigma_i = |lam_i| sorted, Z = Q V_k.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import binding
from .binding import Operator


@dataclass
class KrylovResult:
    sigma: torch.Tensor       # k singular values, nonincreasing (fp64)
    Z: torch.Tensor           # n x k orthonormal columns (top-k Ritz vectors)
    lam: torch.Tensor         # the k signed Ritz values (eigenvalues of A)
    products: int             # number of block products A·(n x b)
    columns: int              # number of fp32 columns through the product (2b per product)
    info: dict = field(default_factory=dict)


def krylov_params(n: int, k: int, block: Optional[int] = None, depth: Optional[int] = None,
                  eps: float = 0.5) -> tuple[int, int]:
    """(b, q): block b = k + 8 and depth q = max(4, ceil(log(n) / sqrt(eps))) by default
    (SPEC S:343), capped so that the basis (q b columns) fits in n and 4096, and b <= 96."""
    if not (1 <= k < n):
        raise ValueError(f"need 1 <= k < n (k={k}, n={n})")
    b = block or min(n, k + 8)
    if not (k <= b <= 96):
        raise ValueError(f"need k <= block <= 96 (k={k}, block={b})")
    q = depth or max(4, math.ceil(math.log(max(n, 2)) / math.sqrt(eps)))
    q = max(1, min(q, n // b, 4096 // b))
    return b, q


def block_krylov(op: Operator, k: int, *, block: Optional[int] = None,
                 depth: Optional[int] = None, eps: float = 0.5, seed: int = 0,
                 start: Optional[torch.Tensor] = None) -> KrylovResult:
    """Top-k singular values / vectors of the symmetric A behind `op` (binding.Operator).
    `start` overrides the Gaussian start block Pi (n x b fp64, seeded from `seed`)."""
    n = op.n
    b, q = krylov_params(n, k, block, depth, eps)
    if start is None:
        gen = torch.Generator(device=op.device).manual_seed(seed)
        start = torch.randn((n, b), generator=gen, dtype=torch.float64, device=op.device)
    sigma, lam, Z, info = binding.l1dm_block_krylov(op, k, start.to(op.device, torch.float64),
                                                    q)
    return KrylovResult(sigma=sigma, Z=Z, lam=lam, products=info["products"],
                        columns=info["columns"], info=info)


def fp64_product(op: Operator, V: torch.Tensor) -> torch.Tensor:
    """A·V for an fp64 block: V = hi + lo (fp32 halves) through one product of width 2b."""
    return binding.l1dm_op_apply(op, V)


def lowrank_error(op: Operator, Z: torch.Tensor, probes: int = 16, seed: int = 1) -> float:
    """Hutchinson estimate of ||A (I - Z Z^T)||_F^2 with `probes` Gaussian vectors (products
    with A only): E ||A (I - Z Z^T) g||^2 = ||A (I - Z Z^T)||_F^2."""
    n = Z.shape[0]
    gen = torch.Generator(device=Z.device).manual_seed(seed)
    G = torch.randn((n, probes), generator=gen, dtype=torch.float64, device=Z.device)
    C = binding.l1dm_gemm(Z, G, trans_a=True)                  # Z^T G
    P = binding.l1dm_gemm(Z, C, G.clone(), alpha=-1.0, beta=1.0)  # G - Z (Z^T G)
    AP = fp64_product(op, P)
    F = binding.l1dm_gemm(AP, AP, trans_a=True)                # (AP)^T AP: its trace
    return float(torch.diagonal(F).sum()) / probes


@dataclass
class CGResult:
    x: torch.Tensor
    iterations: int
    residual: float             # ||A x - b|| / ||b||
    converged: bool
    products: int = 0


def cg_solve(op: Operator, b: torch.Tensor, *, tol: float = 1e-8, maxit: int = 500,
             normal_equations: bool = False) -> CGResult:
    """Conjugate gradients for A x = b with A symmetric positive definite (Thm. linear_system,
    P:741-748), one product per iteration, all scalars on the device.  normal_equations=True
    solves A^2 x = A b (two products per iteration) for symmetric indefinite A such as l1
    distance matrices.  Non-convergence after maxit is reported (converged=False),
    never silent."""
    x, info = binding.l1dm_cg(op, b.to(op.device, torch.float64), tol=tol, maxit=maxit,
                              normal_equations=normal_equations)
    return CGResult(x=x, iterations=int(info["iterations"]), residual=float(info["residual"]),
                    converged=bool(info["converged"]), products=int(info["products"]))
