import sys, numpy as np, torch
import paper_2210_15114_b200 as l1
rng = np.random.default_rng(0)
for (n, d, m, mode) in [(5000, 5, 3, "gather"), (3000, 4, 9, "scatter"), (2000, 3, 1, "auto"), (4000, 3, 2, "auto")]:
    X = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
    if mode == "auto" and m == 2:
        X = torch.floor(X * 3)
    Z = torch.from_numpy(rng.standard_normal((n, m)).astype(np.float32)).cuda()
    h = l1.l1dm_prepare(X)
    if mode != "auto":
        l1.l1dm_set_query_mode(h, mode)
    Y = l1.l1dm_matvec(h, Z)
    Y3 = l1.l1dm_matvec_lp(h, 3, Z)
    torch.cuda.synchronize()
    l1.l1dm_free(h)
print("ok")
