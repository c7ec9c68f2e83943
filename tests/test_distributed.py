"""Coordinate-sharding host logic on CPU with gloo, world size 2.

The local compute is injected from the oracle (the product path has no CPU compute), so
these tests check the partition of coordinates, the per-shard partial products and the
cross-rank SUM (reduce to root and all-reduce) — on integer data, exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2210_15114_b200.distributed import ShardedL1DM, shard_range


def test_shard_range_partitions_coordinates():
    for d in (1, 2, 7, 16, 96, 128):
        for G in (1, 2, 3, 4, 8):
            ranges = [shard_range(d, g, G) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == d
            for (a, b), (c, e) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


class OracleShard:
    """Stand-in for the C-ABI handle: Alg. 1 tables of the full X, Alg. 2 over [k0, k1)."""

    def __init__(self, X, k0, k1):
        self.X = X.numpy()
        self.k0, self.k1 = k0, k1
        _, self.order = oracle.alg1(self.X)


def oracle_prepare(X, k0, k1, stream=None):
    return OracleShard(X, k0, k1)


def oracle_matvec(h, Z, Y=None, stream=None):
    out = torch.from_numpy(oracle.alg2_range(h.X, h.order, h.k0, h.k1, Z.numpy()))
    if Y is not None:
        Y.copy_(out)
        return Y
    return out


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, d, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        X = torch.from_numpy(rng.integers(0, 7, size=(300, d)).astype(np.float32))
        Z = torch.from_numpy(rng.integers(-3, 4, size=(300, 4)).astype(np.float32))
        sh = ShardedL1DM(X, local_prepare=oracle_prepare, local_matvec=oracle_matvec)
        Yr = sh.matvec(Z.clone(), root=0)            # reduce to rank 0
        Ya = sh.matvec(Z.clone(), root=None)         # all-reduce
        part = sh.partial(Z.clone())
        results[rank] = (sh.k_begin, sh.k_end, Yr.numpy().copy(), Ya.numpy().copy(),
                         part.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d", [5, 1])
def test_two_rank_gloo_reduce_and_allreduce(d):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), d, results), nprocs=world, join=True)
    rng = np.random.default_rng(123)
    X = rng.integers(0, 7, size=(300, d)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(300, 4)).astype(np.float32)
    whole = oracle.hist(X, Z, M=6).astype(np.float64)
    (a0, b0, Yr0, Ya0, p0), (a1, b1, Yr1, Ya1, p1) = results[0], results[1]
    assert (a0, b1) == (0, d) and b0 == a1
    assert np.array_equal(Yr0, whole)                 # root holds the sum
    assert np.array_equal(Ya0, whole) and np.array_equal(Ya1, whole)
    assert np.array_equal(p0 + p1, whole)             # partials are the coordinate shares
    if b0 > a0:
        assert np.array_equal(p0, oracle.hist(X[:, a0:b0], Z, M=6).astype(np.float64))
    else:
        assert np.all(p0 == 0)                        # more ranks than coordinates


def lp_worker(rank, world, port, p, results):
    """Odd-p l_p^p (NEXT-1) and even-p (NEXT-4) share the coordinate sharding: A = sum_k A^(k)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        X = torch.from_numpy(rng.integers(0, 5, size=(200, 5)).astype(np.float32))
        Z = torch.from_numpy(rng.integers(-2, 3, size=(200, 3)).astype(np.float32))

        def prep(X_, k0, k1, stream=None):
            return X_[:, k0:k1].contiguous().numpy()

        def mv(h, Z_, Y=None, stream=None):
            return torch.from_numpy(oracle.lp_sorted(h, Z_.numpy(), p) if p % 2
                                    else oracle.lp_even(h, Z_.numpy(), p))

        sh = ShardedL1DM(X, local_prepare=prep, local_matvec=mv, p=p)
        results[rank] = sh.matvec(Z.clone(), root=None).numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [3, 2])
def test_two_rank_gloo_lp(p):
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port = free_port()
    ctx_procs = [ctx.Process(target=lp_worker, args=(r, 2, port, p, results)) for r in range(2)]
    for pr in ctx_procs:
        pr.start()
    for pr in ctx_procs:
        pr.join(120)
        assert pr.exitcode == 0
    rng = np.random.default_rng(7)
    X = rng.integers(0, 5, size=(200, 5)).astype(np.float32)
    Z = rng.integers(-2, 3, size=(200, 3)).astype(np.float32)
    want = oracle.brute_lp(X, Z, p)
    for r in range(2):
        assert np.array_equal(results[r], want)


# ---------------------------------------------------------------- peer-sum buffer exchange
class FakeIPC:
    """Stands in for l1dm_ipc_* on CPU: 'pointers' are integers, a handle names its owner."""

    def __init__(self, rank):
        self.rank, self.count, self.opened, self.closed, self.freed = rank, 0, [], [], []

    def alloc(self, nbytes):
        self.count += 1
        ptr = 1_000_000 * (self.rank + 1) + self.count
        return ptr, f"{ptr}:{nbytes}".encode().ljust(64, b"\0")

    def open(self, handle):
        ptr = int(handle.rstrip(b"\0").split(b":")[0])
        self.opened.append(ptr)
        return ptr + 7  # a mapping is a different address of the same buffer

    def close(self, ptr):
        self.closed.append(ptr)

    def free(self, ptr):
        self.freed.append(ptr)


def peer_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_15114_b200.distributed import PeerGroup, peer_rows
        ipc = FakeIPC(rank)
        n, m = 1001, 3
        pg = PeerGroup(n, m, result_ranks=(0, 2), ipc=ipc)
        pt = pg.peers
        own = {k: (v[0] if v else None) for k, v in pg.own.items()}
        rows = [peer_rows(n, world, o) for o in range(world)]
        out = {
            "world_rank": (pt.world, pt.rank), "inbox": list(pt.inbox[:world]),
            "flags": list(pt.flags[:world]), "ybuf": list(pt.ybuf[:world]),
            "timeout": pt.timeout, "own": own, "mask": pg.targets_mask(), "rows": rows,
            "inbox_bytes": int(pg.own["inbox"][1].rstrip(b"\0").split(b":")[1]),
        }
        pg.close()
        out["closed"] = sorted(ipc.closed)
        out["opened"] = sorted(ipc.opened)
        out["freed"] = sorted(ipc.freed)
        results[rank] = out  # (a manager dict stores copies: assign once, complete)
    finally:
        dist.destroy_process_group()


def test_peer_group_exchange_three_ranks():
    """Every rank maps every other rank's inbox, flags and (result ranks only) result buffer;
    its own buffers stay unmapped; owners' rows partition [0, n); close() unmaps and frees."""
    world = 3
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    mp.start_processes(peer_worker, args=(world, free_port(), results), nprocs=world, join=True,
                       start_method="spawn")
    r = {g: results[g] for g in range(world)}
    assert r[0]["rows"] == [(0, 333), (333, 667), (667, 1001)]
    for g in range(world):
        assert r[g]["world_rank"] == (world, g) and r[g]["mask"] == 0b101
        assert r[g]["timeout"] == r[g]["own"]["timeout"]
        lo, hi = r[g]["rows"][g]
        assert r[g]["inbox_bytes"] == 2 * world * (hi - lo) * 3 * 8  # two epoch halves
        for o in range(world):
            for key in ("inbox", "flags"):
                want = r[o]["own"][key] if o == g else r[o]["own"][key] + 7
                assert r[g][key][o] == want
            if o in (0, 2):
                want = r[o]["own"]["ybuf"] if o == g else r[o]["own"]["ybuf"] + 7
                assert r[g]["ybuf"][o] == want
            else:
                assert r[g]["ybuf"][o] is None
        assert [p + 7 for p in r[g]["opened"]] == r[g]["closed"]
        assert len(r[g]["freed"]) == (4 if g in (0, 2) else 3)
