"""The peer-memory sum of the coordinate shards' partials (l1dm_matvec_push / l1dm_peer_reduce /
l1dm_peer_wait) on one GPU.

Emulation: G ranks live in one process on cuda:0; every rank's push is issued before any
reduce and every reduce before any wait, so no kernel ever waits on another (flags are already
raised when a wait starts).  The peers' buffers are plain local allocations, so the fused
peer-store epilogues, the owner sums and the flag protocol run exactly as across GPUs.  Several
consecutive epochs exercise the double-buffered inboxes.  Reference: the single-handle
l1dm_matvec (same kernels, no sharding) and the CPU oracle; integer data must match exactly.

IPC: two processes map each other's buffers through CUDA IPC handles exchanged over gloo
(PeerGroup) and run the three phases with host barriers between them (again: no waits)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import binding
from paper_2210_15114_b200.distributed import PeerGroup, peer_rows, shard_range

pytestmark = pytest.mark.gpu


class EmulatedGroup:
    """G ranks' peer buffers in one process (all local device memory)."""

    def __init__(self, G, n, m, results):
        self.G, self.n, self.m, self.results = G, n, m, results
        self.bufs = []
        for g in range(G):
            r0, r1 = peer_rows(n, G, g)
            b = {"inbox": binding.l1dm_ipc_alloc(max(2 * G * (r1 - r0) * m * 8, 8))[0],
                 "flags": binding.l1dm_ipc_alloc(2 * G * 4)[0],
                 "timeout": binding.l1dm_ipc_alloc(4)[0],
                 "ybuf": binding.l1dm_ipc_alloc(n * m * 8)[0] if g in results else None}
            self.bufs.append(b)
        self.peers = []
        for g in range(G):
            pt = binding.PeerT()
            pt.world, pt.rank = G, g
            pt.n, pt.m = n, m
            for o in range(G):
                pt.inbox[o] = self.bufs[o]["inbox"]
                pt.flags[o] = self.bufs[o]["flags"]
                pt.ybuf[o] = self.bufs[o]["ybuf"]
            pt.timeout = self.bufs[g]["timeout"]
            self.peers.append(pt)

    def free(self):
        torch.cuda.synchronize()
        for b in self.bufs:
            for v in b.values():
                if v:
                    binding.l1dm_ipc_free(v)


def run_epochs(X, Zs, G, results, mode="auto", ws_limit=0):
    n, d = X.shape
    m = Zs[0].shape[1]
    hs = []
    for g in range(G):
        k0, k1 = shard_range(d, g, G)
        h = l1.l1dm_prepare(X, k0, k1)
        if mode != "auto":
            l1.l1dm_set_query_mode(h, mode)
        if ws_limit:
            l1.l1dm_set_workspace_limit(h, ws_limit)
        hs.append(h)
    grp = EmulatedGroup(G, n, m, results)
    outs = []
    try:
        for e, Z in enumerate(Zs, start=1):
            for g in range(G):
                binding.l1dm_matvec_push(hs[g], Z, grp.peers[g], e)
            for g in range(G):
                binding.l1dm_peer_reduce(grp.peers[g], n, m, e, sum(1 << t for t in results))
            Ys = {}
            for t in results:
                Ys[t] = torch.empty((n, m), dtype=torch.float64, device="cuda")
                binding.l1dm_peer_wait(grp.peers[t], e, n, m, Ys[t])
            for g in range(G):
                binding.l1dm_peer_check(grp.peers[g])
            outs.append({t: Y.cpu().numpy() for t, Y in Ys.items()})
    finally:
        grp.free()
        for h in hs:
            l1.l1dm_free(h)
    return outs


def full_matvec(X, Z, mode="auto"):
    h = l1.l1dm_prepare(X)
    if mode != "auto":
        l1.l1dm_set_query_mode(h, mode)
    Y = l1.l1dm_matvec(h, Z)
    torch.cuda.synchronize()
    l1.l1dm_free(h)
    return Y.cpu().numpy()


@pytest.mark.parametrize("G", [1, 2, 3, 5])
@pytest.mark.parametrize("mode,m", [("gather", 5), ("gather", 1), ("scatter", 12),
                                    ("scatter", 1), ("auto", 3)])
def test_peer_sum_integer_exact(G, mode, m):
    """Integer data: every partial and the sum are exact, so Y must equal the oracle bit for bit
    (gather: fused k6 push; scatter m > 1: fused k9 push; m = 1 scatter: local + k30 push)."""
    rng = np.random.default_rng(100 * G + m)
    n, d = 2500, 11
    Xn = rng.integers(0, 13, size=(n, d)).astype(np.float32)
    X = torch.from_numpy(Xn).cuda()
    Zs = [torch.from_numpy(rng.integers(-4, 5, size=(n, m)).astype(np.float32)).cuda()
          for _ in range(3)]
    results = (0,) if G == 1 else (0, G - 1)
    outs = run_epochs(X, Zs, G, results, mode=mode)
    for Z, out in zip(Zs, outs):
        Yr = oracle.brute(Xn, Z.cpu().numpy())
        for t in results:
            assert np.array_equal(out[t], Yr), (G, mode, m, t)


@pytest.mark.parametrize("G", [2, 4])
def test_peer_sum_chunked_gather_and_runs(G):
    """Gather mode over several coordinate chunks (the last chunk's k6 pushes), and runs mode
    (tie-heavy data: computed locally, pushed by k30)."""
    rng = np.random.default_rng(7 + G)
    n, d, m = 4000, 16, 4
    Xn = rng.integers(0, 6, size=(n, d)).astype(np.float32)
    X = torch.from_numpy(Xn).cuda()
    Zs = [torch.from_numpy(rng.integers(-2, 3, size=(n, m)).astype(np.float32)).cuda()
          for _ in range(2)]
    Yr = [oracle.brute(Xn, Z.cpu().numpy()) for Z in Zs]
    # workspace for ~1 coordinate's U per chunk -> every shard runs several chunks
    outs = run_epochs(X, Zs, G, (0,), mode="gather", ws_limit=n * m * 8 * 3)
    for out, y in zip(outs, Yr):
        assert np.array_equal(out[0], y)
    outs = run_epochs(X, Zs, G, (0,), mode="auto")  # <= 256 distinct values: runs mode
    for out, y in zip(outs, Yr):
        assert np.array_equal(out[0], y)


@pytest.mark.parametrize("m", [1, 16])
def test_peer_sum_float_large_scatter(m):
    """Float data at a scatter-mode size (n >= 2^17): the peer sum against the single handle."""
    rng = np.random.default_rng(m)
    n, d, G = 140000, 12, 3
    X = torch.from_numpy(rng.uniform(-1, 1, size=(n, d)).astype(np.float32)).cuda()
    Zs = [torch.from_numpy(rng.standard_normal((n, m)).astype(np.float32)).cuda()
          for _ in range(2)]
    outs = run_epochs(X, Zs, G, tuple(range(G)))
    for Z, out in zip(Zs, outs):
        Yf = full_matvec(X, Z)
        for t in range(G):
            num = np.linalg.norm(out[t] - Yf, axis=0)
            den = np.maximum(np.linalg.norm(Yf, axis=0), 1e-300)
            assert (num / den).max() <= 1e-12


def test_peer_args_rejected():
    X = torch.rand(100, 3, device="cuda")
    h = l1.l1dm_prepare(X)
    try:
        grp = EmulatedGroup(2, 100, 2, (0,))
        Z = torch.rand(100, 2, device="cuda")
        with pytest.raises(binding.L1dmError):
            binding.l1dm_matvec_push(h, Z, grp.peers[0], 0)  # epoch 0 is reserved
        bad = binding.PeerT()
        bad.world, bad.rank = 2, 5
        with pytest.raises(binding.L1dmError):
            binding.l1dm_matvec_push(h, Z, bad, 1)
        with pytest.raises(binding.L1dmError):  # rank 1 has no result buffer
            binding.l1dm_peer_reduce(grp.peers[0], 100, 2, 1, 0b10)
        # n or m differing from the inbox geometry would store past the owners' slots
        Z3 = torch.rand(100, 3, device="cuda")
        with pytest.raises(binding.L1dmError):
            binding.l1dm_matvec_push(h, Z3, grp.peers[0], 1)
        with pytest.raises(binding.L1dmError):
            binding.l1dm_peer_reduce(grp.peers[0], 101, 2, 1, 0b01)
        with pytest.raises(binding.L1dmError):
            binding.l1dm_peer_wait(grp.peers[0], 1, 100, 3)
        grp.free()
    finally:
        l1.l1dm_free(h)


# ------------------------------------------------------------------ two processes, CUDA IPC
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ipc_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        n, d, m = 3000, 9, 6
        Xn = rng.integers(0, 10, size=(n, d)).astype(np.float32)
        X = torch.from_numpy(Xn).cuda()
        k0, k1 = shard_range(d, rank, world)
        h = l1.l1dm_prepare(X, k0, k1)
        l1.l1dm_set_query_mode(h, "gather")
        pg = PeerGroup(n, m, result_ranks=(0, 1))
        got = []
        for e in (1, 2, 3):
            Z = torch.from_numpy(rng.integers(-3, 4, size=(n, m)).astype(np.float32)).cuda()
            binding.l1dm_matvec_push(h, Z, pg.peers, e)
            torch.cuda.synchronize()
            dist.barrier()  # every arrival flag is up before any reduce starts
            binding.l1dm_peer_reduce(pg.peers, n, m, e, pg.targets_mask(),
                                     stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            dist.barrier()  # every result flag is up before any wait starts
            Y = torch.empty((n, m), dtype=torch.float64, device="cuda")
            binding.l1dm_peer_wait(pg.peers, e, n, m, Y)
            binding.l1dm_peer_check(pg.peers)
            got.append(bool(np.array_equal(Y.cpu().numpy(), oracle.brute(Xn, Z.cpu().numpy()))))
            dist.barrier()
        pg.close()
        l1.l1dm_free(h)
        results[rank] = got
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_peer_sum():
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    mp.start_processes(ipc_worker, args=(2, free_port(), results), nprocs=2, join=True,
                       start_method="spawn")
    assert results[0] == [True] * 3 and results[1] == [True] * 3


def test_peer_sum_more_ranks_than_rows():
    """G = 5 ranks over n = 3 points: two owners hold no rows (empty inbox slots, reduce kernels
    that only wait for their flags); the sum is still exact."""
    rng = np.random.default_rng(3)
    n, d, m, G = 3, 7, 2, 5
    Xn = rng.integers(0, 4, size=(n, d)).astype(np.float32)
    X = torch.from_numpy(Xn).cuda()
    Zs = [torch.from_numpy(rng.integers(-2, 3, size=(n, m)).astype(np.float32)).cuda()]
    outs = run_epochs(X, Zs, G, (0, 4), mode="gather")
    want = oracle.brute(Xn, Zs[0].cpu().numpy())
    assert np.array_equal(outs[0][0], want) and np.array_equal(outs[0][4], want)
