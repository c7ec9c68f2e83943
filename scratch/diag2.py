import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
name = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != '-' else None
w = wl.workload(name, n=n)
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
rows = np.array(sorted(set(np.random.default_rng(0).integers(0, w.n, 8).tolist()) | {0, w.n - 1}))
Yr = oracle.rows(X.cpu().numpy(), Z.cpu().numpy(), rows)
def err(Y):
    Yg = Y[torch.from_numpy(rows).cuda()].cpu().numpy()
    return max(np.linalg.norm(Yg[:, c] - Yr[:, c]) / np.linalg.norm(Yr[:, c]) for c in range(w.m))
h = l1.l1dm_prepare(X)
for q in range(4):
    wb = l1.l1dm_workspace_bytes(h, w.m)
    Y = l1.l1dm_matvec(h, Z); torch.cuda.synchronize()
    try:
        l1.l1dm_sync(h); st = "ok"
    except Exception as e:
        st = str(e)
    print(name, "query", q, "ws", wb, "err %.3e" % err(Y), st, flush=True)
    if q == 1: time.sleep(2)
