import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, paper_2210_15114_b200 as l1
from conftest import col_rel_l2
for (n, d, m) in [(1029, 3, 16), (5000, 2, 16), (3000, 2, 8), (3000, 2, 32), (3000, 2, 64), (3000,2,4), (3000,2,1), (3000,2,2)]:
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d)).astype(np.float32); Z = rng.standard_normal((n, m)).astype(np.float32)
    h = l1.l1dm_prepare(torch.from_numpy(X).cuda())
    Y = l1.l1dm_matvec(h, torch.from_numpy(Z).cuda())
    try:
        torch.cuda.synchronize()
        print(n, d, m, "err", col_rel_l2(Y.cpu().numpy(), oracle.brute(X, Z)), flush=True)
    except Exception as e:
        print(n, d, m, "FAIL", str(e)[:80], flush=True); break
