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


def krylov_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_15114_b200.distributed import ShardedL1DM
        rng = np.random.default_rng(17)
        X = torch.from_numpy(rng.standard_normal((1500, 6)).astype(np.float32)).cuda()
        sh = ShardedL1DM(X, stream=torch.cuda.current_stream())
        r = sh.krylov(6, seed=3)
        # CG on A^2 x = A b converges in O(cond(A)) iterations: a small system (as the one-GPU
        # test, tests/test_gpu_krylov.py::test_cg_normal_equations_on_l1_matrix)
        X2 = torch.from_numpy(rng.standard_normal((150, 4)).astype(np.float32)).cuda()
        sh2 = ShardedL1DM(X2, stream=torch.cuda.current_stream())
        b = torch.from_numpy(rng.standard_normal(150)).cuda()
        c = sh2.cg(b, tol=1e-9, maxit=5000, normal_equations=True)
        torch.cuda.synchronize()
        sh2.close()
        results[rank] = (r.sigma.cpu().numpy().copy(), r.lam.cpu().numpy().copy(),
                         float(c.residual), int(c.iterations), r.products)
        sh.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_sharded_krylov_and_cg():
    """NEXT-2 over coordinate shards: the products are partial A^(K_g) V plus an all-reduce
    (l1dm_block_krylov_cb / l1dm_cg_cb), every dense step in the library on both ranks; the top
    singular values equal numpy.linalg.eigh of the oracle's dense A, identically on both ranks."""
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port = free_port()
    procs = [ctx.Process(target=krylov_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    rng = np.random.default_rng(17)
    X = rng.standard_normal((1500, 6)).astype(np.float32)
    A = oracle.brute(X, np.eye(1500, dtype=np.float32))
    sv = np.sort(np.abs(np.linalg.eigvalsh(A)))[::-1][:6]
    s0, l0, res0, it0, prod0 = results[0]
    s1, l1_, res1, it1, prod1 = results[1]
    assert np.allclose(s0, sv, rtol=1e-8)
    assert np.array_equal(s0, s1) and np.array_equal(l0, l1_)   # identical on every rank
    assert res0 <= 1e-6 and it0 == it1 and prod0 == prod1
