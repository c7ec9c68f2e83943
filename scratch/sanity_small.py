import sys, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import oracle, paper_2210_15114_b200 as l1
from conftest import col_rel_l2
worst = 0.0
for (n, d, m) in [(1, 1, 1), (2, 3, 1), (37, 2, 3), (2049, 2, 1), (700, 3, 16), (513, 2, 64), (300, 2, 65), (1029, 3, 32), (5000, 2, 2)]:
    rng = np.random.default_rng(n + m)
    X = rng.standard_normal((n, d)).astype(np.float32); Z = rng.standard_normal((n, m)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    Y = l1.l1dm_matvec(h, torch.from_numpy(Z).cuda()); torch.cuda.synchronize(); l1.l1dm_sync(h)
    Yr = oracle.brute(X, Z)
    e = 0.0 if n == 1 else col_rel_l2(Y.cpu().numpy(), Yr)
    worst = max(worst, e)
    l1.l1dm_free(h)
print("worst", worst)
