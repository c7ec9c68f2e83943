"""Matrix-free consumers of the block product (PAPER.md §"Applications",
P:727-817): randomized block Krylov for the top-k singular values / a rank-k approximation
(Thm. musco P:735-739 and Thm. bakshi22 P:727-731 as used by Thm. opt_lowrank_p, P:757-766;
SPEC S:340-357) and conjugate gradients (Thm. linear_system).

The only access to A is the block product `matvec(Z) -> A Z` (n x b in, n x b fp64 out): on
the GPU that is this package's C-ABI library (l1dm_matvec, l1dm_matvec_lp,
l1dm_lpp_even_matvec, l1dm_bilinear_matvec ...); the dense steps between products are small
fp64 GEMMs on n x b blocks and a (q b) x (q b) symmetric eigenproblem, done with torch on the
same device (library GEMM / LAPACK-class routines, not the hot path).  Any callable works,
which is how the CPU tests inject a dense or oracle product.

Block Krylov (Musco & Musco's block Krylov iteration for symmetric A, whose singular values
are |eigenvalues|):
  K = [A Pi, A^2 Pi, ..., A^q Pi]  built block by block, each new block orthonormalised
  against all previous ones (block Lanczos without the three-term shortcut: full
  re-orthogonalisation, two passes of classical Gram-Schmidt + CholeskyQR2 inside the block);
  Rayleigh-Ritz: T = Q^T (A Q), T = V diag(lam) V^T, sigma_i = |lam_i| sorted, Z = Q V_k.
A Q costs no extra products: A Q_j is the next block's raw Krylov vector, except for the last
block, which takes one more product.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import torch

MatVec = Callable[[torch.Tensor], torch.Tensor]


@dataclass
class KrylovResult:
    sigma: torch.Tensor       # k singular values, nonincreasing (fp64)
    Z: torch.Tensor           # n x k orthonormal columns (top-k Ritz vectors)
    lam: torch.Tensor         # the k signed Ritz values (eigenvalues of A)
    products: int             # number of block products A·(n x b)
    columns: int              # number of single-vector products (sum of block widths)


def _project_out(V: torch.Tensor, basis: list[torch.Tensor]) -> torch.Tensor:
    """V minus its projection on the span of the (orthonormal) blocks: two passes of block
    classical Gram-Schmidt against the concatenated basis (one pair of GEMMs per pass)."""
    if not basis:
        return V
    B = basis[0] if len(basis) == 1 else torch.cat(basis, dim=1)
    for _ in range(2):
        V = V - B @ (B.T @ V)
    return V


def _eig_orth(V: torch.Tensor, floor: float) -> torch.Tensor:
    """Orthonormal basis of V's column space, dropping directions with singular value <= floor
    (eigen-decomposition of the Gram matrix, applied twice for accuracy)."""
    for rep in range(2):
        G = V.T @ V
        lam, W = torch.linalg.eigh(0.5 * (G + G.T))
        keep = lam > (floor * floor if rep == 0 else 0.25)
        V = V @ (W[:, keep] / torch.sqrt(lam[keep]))
    return V


def _orth_block(V: torch.Tensor, basis: list[torch.Tensor], gen, rtol: float = 1e-9):
    """Orthonormalise V against the previous blocks and within itself.  Directions that lost
    rank (singular value below rtol of V's largest column norm before projection — the Krylov
    space is exhausted, e.g. A of low rank) are re-drawn as fresh Gaussian directions (SPEC
    S:346).  Returns Q (width <= V's), or None when nothing is left (dim reached n)."""
    n, b = V.shape
    scale = float(torch.linalg.norm(V, dim=0).max())
    Q = _eig_orth(_project_out(V, basis), rtol * max(scale, 1e-300))
    have = sum(B.shape[1] for B in basis) + Q.shape[1]
    lost = min(b - Q.shape[1], n - have)
    if lost > 0:
        R = torch.randn((n, lost), generator=gen, dtype=V.dtype, device=gen.device)
        R = _project_out(R, basis + [Q])
        Qr = _eig_orth(R, rtol * float(torch.linalg.norm(R, dim=0).max()))
        Q = torch.cat([Q, Qr], dim=1)
    return Q if Q.shape[1] else None


def fp64_product(matvec: MatVec, V: torch.Tensor, split: bool = True) -> torch.Tensor:
    """A·V for an fp64 block through an fp32-input product: V = hi + lo with hi = fp32(V) and
    lo = fp32(V - hi), one product on the 2b-column block [hi | lo] (linearity), so the result
    carries ~2^-48 relative input rounding instead of fp32's 2^-24.  split=False: fp32(V) only."""
    hi = V.to(torch.float32)
    if not split:
        return matvec(hi.contiguous()).to(V.dtype)
    lo = (V - hi.to(V.dtype)).to(torch.float32)
    out = matvec(torch.cat([hi, lo], dim=1).contiguous()).to(V.dtype)
    b = V.shape[1]
    return out[:, :b] + out[:, b:]


def block_krylov(matvec: MatVec, n: int, k: int, *, block: Optional[int] = None,
                 depth: Optional[int] = None, eps: float = 0.5, seed: int = 0,
                 device=None, dtype=torch.float64, start: Optional[torch.Tensor] = None,
                 split: bool = True) -> KrylovResult:
    """Top-k singular values / vectors of a symmetric A given only `matvec`.

    block b = k + 8 and depth q = max(4, ceil(log(n) / sqrt(eps))) by default.
    matvec receives an fp32 block (the library's query type) and returns A·block in fp64;
    with split=True (default) each fp64 block goes through it as [hi | lo] fp32 halves (one
    product of width 2b), see fp64_product.  `start` overrides the Gaussian start block Pi
    (n x b, seeded from `seed`)."""
    if not (1 <= k < n):
        raise ValueError(f"need 1 <= k < n (k={k}, n={n})")
    b = block or min(n, k + 8)
    q = depth or max(4, math.ceil(math.log(max(n, 2)) / math.sqrt(eps)))
    gdev = torch.device(device) if device is not None else torch.device("cpu")
    gen = torch.Generator(device=gdev).manual_seed(seed)
    Pi = start if start is not None else torch.randn((n, b), generator=gen, dtype=dtype,
                                                     device=gdev)
    Pi = Pi.to(device=gdev, dtype=dtype)
    products = columns = 0

    def apply(V: torch.Tensor) -> torch.Tensor:
        nonlocal products, columns
        products += 1
        columns += V.shape[1] * (2 if split else 1)
        return fp64_product(matvec, V, split)

    # the basis and A times it live in preallocated n x (q b) buffers (views, no re-concatenation)
    Qbuf = torch.empty((n, q * b), dtype=dtype, device=gdev)
    AQbuf = torch.empty((n, q * b), dtype=dtype, device=gdev)
    cols = 0
    W = apply(Pi)                    # A Pi: the first Krylov block
    for _ in range(q):
        width = min(b, n - cols)
        if width <= 0:
            break
        Q = _orth_block(W[:, :width], [Qbuf[:, :cols]] if cols else [], gen)
        if Q is None:
            break
        w_ = Q.shape[1]
        Qbuf[:, cols:cols + w_] = Q
        W = apply(Q)                 # A Q_j: Rayleigh-Ritz column block and next Krylov block
        AQbuf[:, cols:cols + w_] = W
        cols += w_
    Qm = Qbuf[:, :cols]
    T = Qm.T @ AQbuf[:, :cols]       # Rayleigh quotient Q^T A Q
    T = 0.5 * (T + T.T)
    lam, V = torch.linalg.eigh(T)
    order = torch.argsort(lam.abs(), descending=True)[:k]
    lam_k = lam[order]
    Z = Qm @ V[:, order]
    return KrylovResult(sigma=lam_k.abs(), Z=Z, lam=lam_k, products=products, columns=columns)


def lowrank_error(matvec: MatVec, Z: torch.Tensor, probes: int = 16, seed: int = 1) -> float:
    """Hutchinson estimate of ||A (I - Z Z^T)||_F^2 using `probes` Gaussian vectors (only
    products with A): E ||A (I - Z Z^T) g||^2 = ||A (I - Z Z^T)||_F^2."""
    n = Z.shape[0]
    gen = torch.Generator(device=Z.device).manual_seed(seed)
    G = torch.randn((n, probes), generator=gen, dtype=Z.dtype, device=Z.device)
    P = G - Z @ (Z.T @ G)
    AP = fp64_product(matvec, P)
    return float((AP * AP).sum() / probes)


@dataclass
class CGResult:
    x: torch.Tensor
    iterations: int
    residual: float             # ||A x - b|| / ||b||
    converged: bool


def cg_solve(matvec: MatVec, b: torch.Tensor, *, tol: float = 1e-8, maxit: int = 500,
             normal_equations: bool = False) -> CGResult:
    """Conjugate gradients for A x = b with A symmetric positive definite (Thm. linear_system,
    P:741-748), one product per iteration.  normal_equations=True solves A^2 x = A b (two
    products per iteration) for symmetric indefinite A such as l1 distance matrices.
    Non-convergence after maxit is reported (converged=False), never silent."""
    dtype = torch.float64
    b = b.to(dtype).reshape(-1, 1)

    def A(v):
        return fp64_product(matvec, v.reshape(-1, 1)).reshape(-1, 1)

    def op(v):
        return A(A(v)) if normal_equations else A(v)

    rhs = A(b) if normal_equations else b
    x = torch.zeros_like(b)
    r = rhs.clone()
    p = r.clone()
    rs = float((r * r).sum())
    bn = float(torch.linalg.norm(b))
    target = tol * float(torch.linalg.norm(rhs))
    it, converged = 0, math.sqrt(rs) <= target
    while not converged and it < maxit:
        it += 1
        Ap = op(p)
        alpha = rs / float((p * Ap).sum())
        x = x + alpha * p
        r = r - alpha * Ap
        rs_new = float((r * r).sum())
        converged = math.sqrt(rs_new) <= target
        p = r + (rs_new / rs) * p
        rs = rs_new
    res = float(torch.linalg.norm(A(x) - b)) / max(bn, 1e-300)
    return CGResult(x=x.reshape(-1), iterations=it, residual=res, converged=converged)
