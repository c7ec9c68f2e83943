"""Seeded synthetic inputs for the five BASELINE.json configs (and scaled-down variants).

This module holds RANDOM NUMBER GENERATION ONLY — none of the method's
arithmetic — so that the CUDA path and the CPU oracle can be fed the very same
inputs (the task's "seeded input generators" rule).  It imports neither the
oracle nor the CUDA binding.

Recipe, X drawn first, then Z, each from its own torch.Generator
(Philox on CUDA, the CPU generator on CPU — the device is part of the recipe):

  c1  n=2048,  d=16,  X ~ U[0,1),                      m=1,  Z ~ N(0,1),  seed 0
  c2  n=2^20,  d=64,  X ~ N(0,1),                      m=1,  Z ~ N(0,1),  seed 1
  c3  n=2^20,  d=128, X ~ U[-1,1),                     m=64, Z ~ N(0,1),  seed 2
  c4  n=2^24,  d=128, X ~ 32-cluster GMM: centres U[-10,10]^d (drawn first),
                      equal-weight i.i.d. assignment, x = c_a + 0.5 N(0,I),
                                                       m=32, Z ~ N(0,1),  seed 3
  c5  n=2^23,  d=96,  X = floor(256 U) in {0..255},    m=16, Z ~ U{-1,+1}, seed 4

Fresh query blocks (c2/c4/c5 trials) use seed 1000*c + t for trial t.
Every config can be drawn at a smaller n (and d, m) for parity tests: the value
distribution and structure (ties, clusters) are the config's.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import torch


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    m: int
    x_dist: str          # "uniform01" | "normal" | "uniform11" | "gmm32" | "int256"
    z_dist: str          # "normal" | "pm1"
    seed: int
    queries: int         # queries per step in the bench recipe
    fresh_queries: bool  # True: a new Z per query (seed 1000*c+t); False: one fixed Z

    @property
    def index(self) -> int:
        if self.name.startswith("ctx"):
            return 5 + int(self.name[3:])
        return int(self.name[1:]) if self.name[1:].isdigit() else 9

    @property
    def updates_per_query(self) -> int:
        return self.n * self.d * self.m


CONFIGS = {
    "c1": Workload("c1", 2048, 16, 1, "uniform01", "normal", 0, 20, True),
    "c2": Workload("c2", 1 << 20, 64, 1, "normal", "normal", 1, 20, True),
    "c3": Workload("c3", 1 << 20, 128, 64, "uniform11", "normal", 2, 100, False),
    "c4": Workload("c4", 1 << 24, 128, 32, "gmm32", "normal", 3, 10, True),
    "c5": Workload("c5", 1 << 23, 96, 16, "int256", "pm1", 4, 10, True),
    # SURVEY §8(d) "ctx" (optional): the shapes of the paper's Table 3, synthetic
    # stand-ins, to place B200 times beside the paper's as context only: a 3-cluster Gaussian
    # mixture in R^50, MNIST-like 8-bit integers in R^784 with 80% zeros (assumed: the paper
    # does not describe its data), GloVe-like N(0,1) in R^50; m = 1, 10 Gaussian queries
    "ctx1": Workload("ctx1", 50000, 50, 1, "gmm3", "normal", 5, 10, True),
    "ctx2": Workload("ctx2", 50000, 784, 1, "mnist80", "normal", 6, 10, True),
    "ctx3": Workload("ctx3", 1200000, 50, 1, "normal", "normal", 7, 10, True),
}
# Table 3's "Ours" rows (2021 M1 MacBook Pro, Python + NumPy/Numba):
# (preprocessing s, average query s) — context, not a target
PAPER_TABLE3 = {"ctx1": (0.55, 0.09), "ctx2": (5.5, 1.9), "ctx3": (16.8, 3.4)}


def workload(name: str, n: int | None = None, d: int | None = None, m: int | None = None,
             seed: int | None = None) -> Workload:
    w = CONFIGS[name]
    kw = {}
    if n is not None:
        kw["n"] = int(n)
    if d is not None:
        kw["d"] = int(d)
    if m is not None:
        kw["m"] = int(m)
    if seed is not None:
        kw["seed"] = int(seed)
    return replace(w, **kw) if kw else w


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def make_points(w: Workload, device="cpu") -> torch.Tensor:
    """X: n x d fp32, row-major, on `device`."""
    g = _gen(device, w.seed)
    n, d = w.n, w.d
    if w.x_dist == "uniform01":
        return torch.rand((n, d), generator=g, device=device, dtype=torch.float32)
    if w.x_dist == "normal":
        return torch.randn((n, d), generator=g, device=device, dtype=torch.float32)
    if w.x_dist == "uniform11":
        X = torch.rand((n, d), generator=g, device=device, dtype=torch.float32)
        return X.mul_(2.0).sub_(1.0)
    if w.x_dist == "gmm32":
        centres = torch.rand((32, d), generator=g, device=device, dtype=torch.float32)
        centres.mul_(20.0).sub_(10.0)
        assign = torch.randint(0, 32, (n,), generator=g, device=device)
        X = torch.randn((n, d), generator=g, device=device, dtype=torch.float32)
        X.mul_(0.5)
        X.add_(centres.index_select(0, assign))
        return X
    if w.x_dist == "gmm3":  # 3 spherical clusters, centres U[-10, 10]^d, sigma 0.5 (as c4)
        centres = torch.rand((3, d), generator=g, device=device, dtype=torch.float32)
        centres.mul_(20.0).sub_(10.0)
        assign = torch.randint(0, 3, (n,), generator=g, device=device)
        X = torch.randn((n, d), generator=g, device=device, dtype=torch.float32)
        X.mul_(0.5)
        X.add_(centres.index_select(0, assign))
        return X
    if w.x_dist == "mnist80":  # integers 1..255 with probability 0.2, else 0
        v = torch.rand((n, d), generator=g, device=device, dtype=torch.float32)
        keep = torch.rand((n, d), generator=g, device=device, dtype=torch.float32) < 0.2
        return torch.where(keep, v.mul_(255.0).floor_().add_(1.0).clamp_(1.0, 255.0),
                           torch.zeros_like(v))
    if w.x_dist == "int256":
        X = torch.rand((n, d), generator=g, device=device, dtype=torch.float32)
        return X.mul_(256.0).floor_().clamp_(0.0, 255.0)
    raise ValueError(w.x_dist)


def make_query(w: Workload, trial: int = 0, device="cpu") -> torch.Tensor:
    """Z: n x m fp32, row-major.  Fixed-Z configs ignore `trial`."""
    t = trial if w.fresh_queries else 0
    seed = 1000 * w.index + t + 100003 * (w.seed - CONFIGS[w.name].seed)
    g = _gen(device, seed)
    n, m = w.n, w.m
    if w.z_dist == "normal":
        return torch.randn((n, m), generator=g, device=device, dtype=torch.float32)
    if w.z_dist == "pm1":
        b = torch.randint(0, 2, (n, m), generator=g, device=device, dtype=torch.int32)
        return b.to(torch.float32).mul_(2.0).sub_(1.0)
    raise ValueError(w.z_dist)


def gaussian_embedding(k: int, d: int, seed: int, device="cpu") -> torch.Tensor:
    """G: k x d fp32 of i.i.d. N(0,1) draws — the random matrix of Thm. l2embed,
    passed to both the library (l1dm_l2_embed) and the oracle as an input (RNG only here)."""
    return torch.randn((k, d), generator=_gen(device, 7_000_003 + seed), device=device,
                       dtype=torch.float32)
