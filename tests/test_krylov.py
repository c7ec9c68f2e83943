"""Host logic of the matrix-free consumers: the parameter choice, and that
nothing runs without the library on a GPU (every dense step lives in libl1dm.so, include/l1dm.h
"Matrix-free consumers"; there is no host or torch fallback).  The algorithm itself is checked
on the GPU in test_gpu_krylov.py against numpy.linalg.eigh of the oracle's dense A."""
import math

import pytest
import torch

from paper_2210_15114_b200 import binding
from paper_2210_15114_b200.krylov import krylov_params


def test_default_parameters_follow_spec():
    # block k + 8, depth max(4, ceil(log n / sqrt(eps)))
    n = 1 << 20
    b, q = krylov_params(n, 16, eps=0.5)
    assert b == 24 and q == max(4, math.ceil(math.log(n) / math.sqrt(0.5))) == 20
    assert krylov_params(n, 16, block=32, depth=6) == (32, 6)


def test_parameters_capped_by_n():
    assert krylov_params(120, 1) == (9, 7)
    assert krylov_params(100, 10) == (18, 5)         # q b <= n: 7 * 18 > 100
    assert krylov_params(10, 2) == (10, 1)           # block capped at n
    with pytest.raises(ValueError):
        krylov_params(4, 4)                          # k < n
    with pytest.raises(ValueError):
        krylov_params(1000, 10, block=5)             # block >= k
    with pytest.raises(ValueError):
        krylov_params(10 ** 6, 10, block=128)        # block <= 96


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_fallback_without_gpu():
    A = torch.eye(3, dtype=torch.float64)
    with pytest.raises((binding.L1dmError, ImportError, ValueError)):
        binding.l1dm_gemm(A, A)
    with pytest.raises((binding.L1dmError, ImportError, ValueError)):
        binding.l1dm_syevj(A)
    with pytest.raises(ValueError):
        binding.Operator.bilinear(torch.zeros(4, 2), torch.eye(2, dtype=torch.float64))
