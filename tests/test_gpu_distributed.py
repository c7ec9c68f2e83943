"""The multi-rank query path with the real library on one GPU: two processes (gloo for the
collective, both ranks' kernels on cuda:0 — they never wait on one another), each holding
one coordinate shard; the summed Y must equal the oracle (integer data: exactly).  Covers
ShardedL1DM's plain and point-block-overlapped paths (l1dm_matvec_pipelined + per-block
all-reduce) in both query strategies."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, mode, blocks, root, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_15114_b200.distributed import ShardedL1DM
        rng = np.random.default_rng(5)
        X = torch.from_numpy(rng.integers(0, 9, size=(3000, 7)).astype(np.float32)).cuda()
        Z = torch.from_numpy(rng.integers(-3, 4, size=(3000, 12)).astype(np.float32)).cuda()
        sh = ShardedL1DM(X, stream=torch.cuda.current_stream(), mode=mode)
        Y = sh.matvec(Z, root=root, overlap_blocks=blocks)
        torch.cuda.synchronize()
        results[rank] = Y.cpu().numpy().copy()
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,blocks,root", [("gather", 1, None), ("gather", 4, None),
                                              ("scatter", 1, None), ("scatter", 3, None),
                                              ("gather", 4, 0), ("scatter", 2, 0)])
def test_two_ranks_one_gpu_sum_is_exact(mode, blocks, root):
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, mode, blocks, root, results))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    X = rng.integers(0, 9, size=(3000, 7)).astype(np.float32)
    Z = rng.integers(-3, 4, size=(3000, 12)).astype(np.float32)
    want = oracle.hist(X, Z, M=8).astype(np.float64)
    for r in (range(2) if root is None else [root]):   # reduce: the root holds the sum
        assert np.array_equal(results[r], want)
