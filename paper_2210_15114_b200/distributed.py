"""Coordinate sharding over torch.distributed (one process per GPU; NCCL over NVLink).

A = sum_k A^(k) with A^(k)_ij = |x_ik - x_jk| (the swap of sums in the proof of
Thm "p=1"), so rank g prepares only its coordinate slice K_g and
returns the partial Y_g = A^(K_g) Z (its own share of the g - h S epilogue
included, reading R15).  One fp64 SUM collective combines the partials:
reduce to a root (BASELINE.json north_star "NCCL reduce") or all-reduce when every
rank needs Y (Krylov-style consumers).  Prepare is communication-free.

The local compute is the C ABI (l1dm_prepare_ex / l1dm_matvec_ex).  For host-side
tests of the sharding logic on CPU (gloo), `local_prepare` / `local_matvec` can be
injected; the product default never runs anything but the CUDA library.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import binding


def shard_range(d: int, rank: int, world: int) -> tuple[int, int]:
    """Coordinates [floor(g d / G), floor((g+1) d / G)) for rank g of G."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    return (rank * d) // world, ((rank + 1) * d) // world


class ShardedL1DM:
    """Per-rank handle over a coordinate shard, with the cross-rank sum of Y."""

    def __init__(self, X: torch.Tensor, group=None, *, k_range=None,
                 local_prepare: Optional[Callable] = None,
                 local_matvec: Optional[Callable] = None, stream=None, mode: str = "auto",
                 p: int = 1):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        d = X.shape[1]
        self.k_begin, self.k_end = k_range if k_range is not None else shard_range(
            d, self.rank, self.world)
        if local_matvec is None and p % 2 == 1 and p != 1:  # odd l_p^p (Thm. odd_p): A = sum_k A^(k)
            local_matvec = (lambda h, Z, Y=None, stream=None:
                            binding.l1dm_matvec_lp(h, p, Z, Y, stream=stream))
        if local_prepare is None and p % 2 == 0:  # even p (NEXT-4): sort-free, the "handle" is X_g
            local_prepare = (lambda X_, k0, k1, stream=None: X_[:, k0:k1].contiguous())
            local_matvec = (lambda h, Z, Y=None, stream=None:
                            binding.l1dm_lpp_even_matvec(h, p, Z, Y, stream=stream))
        self._prepare = local_prepare or binding.l1dm_prepare
        self._matvec = local_matvec or binding.l1dm_matvec
        self.stream = stream
        if self.k_end > self.k_begin:
            self.handle = self._prepare(X, self.k_begin, self.k_end, stream=stream)
            if mode != "auto" and self._prepare is binding.l1dm_prepare:
                binding.l1dm_set_query_mode(self.handle, mode)
        else:
            self.handle = None  # more ranks than coordinates: this rank contributes zeros

    def partial(self, Z: torch.Tensor, Y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Y_g = A^(K_g) Z for this rank's coordinates (no communication)."""
        n, m = Z.shape[0], (Z.shape[1] if Z.dim() == 2 else 1)
        if self.handle is None:
            if Y is None:
                Y = torch.zeros((n, m), dtype=torch.float64, device=Z.device)
            else:
                Y.zero_()
            return Y
        return self._matvec(self.handle, Z, Y, stream=self.stream)

    def matvec(self, Z: torch.Tensor, Y: Optional[torch.Tensor] = None, *, root: Optional[int] = 0,
               async_op: bool = False, overlap_blocks: int = 1):
        """A·Z summed over ranks: on `root` only (reduce) or on every rank (root=None).

        overlap_blocks > 1 (CUDA, C-ABI handle): the last accumulate runs per point block and
        each block's rows are reduced as soon as they are final, overlapping the collective with
        the remaining blocks' compute."""
        if (overlap_blocks > 1 and self.world > 1 and self.handle is not None and Z.is_cuda
                and self._matvec is binding.l1dm_matvec):
            return self._matvec_overlapped(Z, Y, root, async_op, overlap_blocks)
        Y = self.partial(Z, Y)
        if self.world == 1:
            return (Y, None) if async_op else Y
        if root is None:
            work = dist.all_reduce(Y, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)
        else:
            work = dist.reduce(Y, dst=root, op=dist.ReduceOp.SUM, group=self.group,
                               async_op=async_op)
        return (Y, work) if async_op else Y

    def _matvec_overlapped(self, Z, Y, root, async_op, nblocks):
        n, m = Z.shape[0], Z.shape[1]
        if Y is None:
            Y = torch.empty((n, m), dtype=torch.float64, device=Z.device)
        main = torch.cuda.current_stream(Z.device)
        if getattr(self, "_compute_stream", None) is None:
            self._compute_stream = torch.cuda.Stream(device=Z.device)
        cs = self._compute_stream
        cs.wait_stream(main)                      # Z (and Y's previous users) are ready
        scatter, mb, ncb = binding.l1dm_query_layout(self.handle, m)
        if scatter and m > 1:
            # scatter strategy: rows are final only after the last column block, so the sum runs
            # per column block of a column-block-major staging copy
            Yb = torch.empty((ncb, n, mb), dtype=torch.float64, device=Z.device)
            events = [torch.cuda.Event() for _ in range(ncb)]
            binding.l1dm_matvec_colblocks(self.handle, Z, Yb, events, stream=cs)
            works = []
            for b, ev in enumerate(events):
                main.wait_event(ev)
                works.append(self._collective(Yb[b], root))
            for w in works:
                w.wait()
            binding.l1dm_unblock(Yb, m, Y, stream=main)
            return (Y, []) if async_op else Y
        events = [torch.cuda.Event() for _ in range(nblocks)]
        binding.l1dm_matvec_pipelined(self.handle, Z, Y, events, stream=cs)
        works = []
        for (i0, i1), ev in zip(binding.point_blocks(n, nblocks), events):
            # the main stream (which NCCL synchronises with) waits only for block b's rows, so
            # block b's collective runs while the compute stream finishes blocks b+1..
            main.wait_event(ev)
            works.append(self._collective(Y[i0:i1], root))
        if async_op:
            return Y, works
        for w in works:
            w.wait()
        return Y

    def _collective(self, T, root):
        if root is None:
            return dist.all_reduce(T, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        return dist.reduce(T, dst=root, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    def close(self):
        if self.handle is not None and self._prepare is binding.l1dm_prepare:
            binding.l1dm_free(self.handle)
        self.handle = None
