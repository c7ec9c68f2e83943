import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
name = sys.argv[1]; reps = int(sys.argv[2])
w = wl.workload(name, n=int(sys.argv[3]) if len(sys.argv) > 3 else None)
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
h = l1.l1dm_prepare(X)
Y0 = l1.l1dm_matvec(h, Z).clone(); torch.cuda.synchronize()
worst = 0.0; bad = 0
for r in range(reps):
    Y = l1.l1dm_matvec(h, Z); torch.cuda.synchronize()
    rel = ((Y - Y0).norm(dim=0) / Y0.norm(dim=0)).max().item()
    worst = max(worst, rel); bad += rel > 1e-12
l1.l1dm_sync(h)
print(name, "reps", reps, "max rel diff between runs", worst, "bad", bad, flush=True)
