import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
from conftest import col_rel_l2
name = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = wl.workload(name, n=n)
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
h = l1.l1dm_prepare(X)
rows = np.array(sorted(set(np.random.default_rng(0).integers(0, w.n, 12).tolist()) | {0, w.n - 1}))
Xh, Zh = X.cpu().numpy(), Z.cpu().numpy()
Yr = oracle.rows(Xh, Zh, rows)
for ws in [0, 8 << 30, 64 << 30]:
    l1.l1dm_set_workspace_limit(h, ws)
    Y = l1.l1dm_matvec(h, Z); torch.cuda.synchronize(); l1.l1dm_sync(h)
    Yg = Y[torch.from_numpy(rows).cuda()].cpu().numpy()
    err = [np.linalg.norm(Yg[:, c] - Yr[:, c]) / np.linalg.norm(Yr[:, c]) for c in range(min(4, w.m))]
    print(name, "ws", ws, "ws_bytes", l1.l1dm_workspace_bytes(h, w.m), "err", err, flush=True)
    print(" gpu", Yg[:3, 0], "\n ref", Yr[:3, 0], flush=True)
    del Y
# sort tables sanity at full size: perm is permutation & sval sorted for a few coords
sval, perm, rank, hs = l1.l1dm_debug_export(h)
for k in [0, 63, 127 if w.d > 127 else w.d - 1]:
    ok1 = np.all(np.diff(sval[k]) >= 0); ok2 = np.array_equal(np.sort(perm[k]), np.arange(w.n, dtype=np.uint32))
    ok3 = np.array_equal(rank[k][perm[k]], np.arange(w.n, dtype=np.uint32)); ok4 = np.array_equal(sval[k], Xh[perm[k], k])
    print("coord", k, ok1, ok2, ok3, ok4, flush=True)
