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


def peer_rows(n: int, world: int, owner: int) -> tuple[int, int]:
    """Rows [floor(o n / G), floor((o+1) n / G)) owned by rank o in the peer sum."""
    return (n * owner) // world, (n * (owner + 1)) // world


class PeerGroup:
    """The symmetric device buffers of the peer-memory sum (include/l1dm.h).

    Every rank allocates its inbox (two epoch-parity halves of G slots of its rows x m fp64), 2G
    flag words, a timeout word
    and, on result ranks, an n x m result buffer with l1dm_ipc_alloc; the CUDA IPC handles are
    exchanged with one all_gather_object and each rank maps every other rank's buffers with
    l1dm_ipc_open.  `ipc` (alloc/open/close/free) can be injected for host-side tests."""

    def __init__(self, n: int, m: int, group=None, *, result_ranks=(0,), ipc=None):
        from types import SimpleNamespace
        ipc = ipc or SimpleNamespace(alloc=binding.l1dm_ipc_alloc, open=binding.l1dm_ipc_open,
                                     close=binding.l1dm_ipc_close, free=binding.l1dm_ipc_free)
        self.ipc, self.n, self.m, self.group = ipc, n, m, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > binding.MAX_PEERS:
            raise ValueError(f"peer sum supports at most {binding.MAX_PEERS} ranks")
        G, g = self.world, self.rank
        self.result_ranks = sorted(set(result_ranks))
        r0, r1 = peer_rows(n, G, g)
        self.own = {"inbox": ipc.alloc(max(2 * G * (r1 - r0) * m * 8, 8)),  # 2 epoch halves
                    "flags": ipc.alloc(2 * G * 4), "timeout": ipc.alloc(4),
                    "ybuf": ipc.alloc(n * m * 8) if g in self.result_ranks else None}
        mine = {k: (v[1] if v else None) for k, v in self.own.items() if k != "timeout"}
        allh = [None] * G
        if G > 1:
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh[0] = mine
        self.mapped = []  # pointers this process opened (closed in close())
        pt = binding.PeerT()
        pt.world, pt.rank = G, g
        pt.n, pt.m = n, m
        for o in range(G):
            for key, arr in (("inbox", pt.inbox), ("flags", pt.flags), ("ybuf", pt.ybuf)):
                if o == g:
                    arr[o] = self.own[key][0] if self.own[key] else None
                elif allh[o][key] is not None:
                    ptr = ipc.open(allh[o][key])
                    self.mapped.append(ptr)
                    arr[o] = ptr
        pt.timeout = self.own["timeout"][0]
        self.peers = pt
        self.epoch = 0

    def targets_mask(self) -> int:
        return sum(1 << t for t in self.result_ranks)

    def close(self):
        for ptr in self.mapped:
            self.ipc.close(ptr)
        self.mapped = []
        for v in self.own.values():
            if v:
                self.ipc.free(v[0])
        self.own = {}


class ShardedL1DM:
    """Per-rank handle over a coordinate shard, with the cross-rank sum of Y."""

    def __init__(self, X: torch.Tensor, group=None, *, k_range=None,
                 local_prepare: Optional[Callable] = None,
                 local_matvec: Optional[Callable] = None, stream=None, mode: str = "auto",
                 p: int = 1, peer_group: Optional["PeerGroup"] = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        d = X.shape[1]
        self.n, self.p = X.shape[0], p
        self.k_begin, self.k_end = k_range if k_range is not None else shard_range(
            d, self.rank, self.world)
        if local_matvec is None and p % 2 == 1 and p != 1:  # odd l_p^p (Thm. odd_p): A = sum_k A^(k)
            local_matvec = (lambda h, Z, Y=None, stream=None:
                            binding.l1dm_matvec_lp(h, p, Z, Y, stream=stream))
        if local_prepare is None and p % 2 == 0:  # even p (NEXT-4): sort-free, the "handle" is X_g
            local_prepare = (lambda X_, k0, k1, stream=None: X_[:, k0:k1].contiguous())
            local_matvec = (lambda h, Z, Y=None, stream=None:
                            binding.l1dm_lpp_even_matvec(h, p, Z, Y, stream=stream))
        self._peer = peer_group      # collective="peer" buffers (reused across handles if given)
        self._peer_owned = peer_group is None
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
               async_op: bool = False, overlap_blocks: int = 1, collective: str = "nccl",
               check: bool = True):
        """A·Z summed over ranks: on `root` only (reduce) or on every rank (root=None).

        overlap_blocks > 1 (CUDA, C-ABI handle): the last accumulate runs per point block and
        each block's rows are reduced as soon as they are final, overlapping the collective with
        the remaining blocks' compute.
        collective="peer" (CUDA, l1 handle): the sum runs over peer memory in this library's
        kernels — the query's final pass stores rows straight into their owners' inboxes
        (l1dm_matvec_push), owners reduce and store into the result ranks (l1dm_peer_reduce),
        result ranks wait (l1dm_peer_wait); no NCCL on the data path.  check=True (default)
        synchronises the stream after the query and raises L1dmError(ETIMEOUT) if any of this
        rank's bounded peer waits gave up (the group is then rebuilt on the next call)."""
        if collective == "peer":
            return self._matvec_peer(Z, Y, root, check)
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

    def _matvec_peer(self, Z, Y, root, check=True):
        if self.handle is None or self._matvec is not binding.l1dm_matvec or not Z.is_cuda:
            raise ValueError("collective='peer' needs a CUDA Z and an l1 C-ABI handle on every rank")
        n, m = Z.shape[0], Z.shape[1]
        results = tuple(range(self.world)) if root is None else (root,)
        pg = getattr(self, "_peer", None)
        if pg is None or pg.m != m or pg.n != n or tuple(pg.result_ranks) != results:
            if pg is not None and self._peer_owned:
                torch.cuda.synchronize(Z.device)
                pg.close()
            pg = self._peer = PeerGroup(n, m, self.group, result_ranks=results)
            self._peer_owned = True
        pg.epoch += 1
        stream = self.stream
        binding.l1dm_matvec_push(self.handle, Z, pg.peers, pg.epoch, stream=stream)
        binding.l1dm_peer_reduce(pg.peers, n, m, pg.epoch, pg.targets_mask(),
                                 stream=stream if stream is not None
                                 else torch.cuda.current_stream(Z.device))
        if self.rank in results:
            if Y is None:
                Y = torch.empty((n, m), dtype=torch.float64, device=Z.device)
            binding.l1dm_peer_wait(pg.peers, pg.epoch, n, m, Y, stream=stream)
        if check:
            # a bounded flag wait that gave up leaves Y invalid: raise instead of returning it,
            # and drop the group — after a timeout the epoch-parity reuse argument is void
            try:
                binding.l1dm_peer_check(pg.peers, stream=stream if stream is not None
                                        else torch.cuda.current_stream(Z.device))
            except binding.L1dmError:
                if self._peer_owned:
                    torch.cuda.synchronize(Z.device)
                    pg.close()
                self._peer = None
                raise
        return Y

    # ---- matrix-free consumers over the shards ("needs all-reduce")
    def _fp64_product(self, V: torch.Tensor, Y: torch.Tensor, stream) -> None:
        """Y = A V for an fp64 block on every rank: this rank's partial A^(K_g) V through the
        library (hi/lo split), then an all-reduce (sum over the coordinate shards)."""
        if self.handle is None:
            part = torch.zeros_like(Y)
        else:
            part = binding.l1dm_op_apply(self._operator(), V, stream=stream)
        if self.world > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
        Y.copy_(part)

    def _operator(self):
        if getattr(self, "_op", None) is None:
            if self._prepare is not binding.l1dm_prepare:
                raise ValueError("the consumers need the library's handle on every rank")
            p = getattr(self, "p", 1)
            self._op = binding.Operator.sorted(self.handle, p)
        return self._op

    def krylov(self, k: int, *, block: Optional[int] = None, depth: Optional[int] = None,
               eps: float = 0.5, seed: int = 0):
        """Top-k singular values of A (Thm. musco) with the products sharded over
        the ranks and all-reduced; every dense step in the library, identical on every rank
        (the same start block from the seed, deterministic kernels, all-reduced products)."""
        from .krylov import KrylovResult, krylov_params
        n = self.n
        b, q = krylov_params(n, k, block, depth, eps)
        dev = torch.device("cuda", torch.cuda.current_device())
        gen = torch.Generator(device=dev).manual_seed(seed)
        Pi = torch.randn((n, b), generator=gen, dtype=torch.float64, device=dev)
        sigma, lam, Z, info = binding.l1dm_block_krylov_cb(
            n, lambda V, Y, st: self._fp64_product(V, Y, st), k, Pi, q)
        return KrylovResult(sigma=sigma, Z=Z, lam=lam, products=info["products"],
                            columns=info["columns"], info=info)

    def cg(self, b: torch.Tensor, *, tol: float = 1e-8, maxit: int = 500,
           normal_equations: bool = False):
        """Conjugate gradients (Thm. linear_system) on the sharded operator."""
        from .krylov import CGResult
        x, info = binding.l1dm_cg_cb(self.n, lambda V, Y, st: self._fp64_product(V, Y, st),
                                     b.to(torch.float64), tol=tol, maxit=maxit,
                                     normal_equations=normal_equations)
        return CGResult(x=x, iterations=int(info["iterations"]), residual=float(info["residual"]),
                        converged=bool(info["converged"]), products=int(info["products"]))

    def _collective(self, T, root):
        if root is None:
            return dist.all_reduce(T, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        return dist.reduce(T, dst=root, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    def close(self):
        if getattr(self, "_peer", None) is not None and self._peer_owned:
            torch.cuda.synchronize()
            self._peer.close()
        self._peer = None
        if self.handle is not None and self._prepare is binding.l1dm_prepare:
            binding.l1dm_free(self.handle)
        self.handle = None
