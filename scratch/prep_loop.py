import sys, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload(sys.argv[1]); X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
Y = torch.empty((w.n, w.m), dtype=torch.float64, device="cuda")
for it in range(4):
    torch.cuda.synchronize()
    print("---- step", it, file=sys.stderr, flush=True)
    h = l1.l1dm_prepare(X)
    l1.l1dm_matvec(h, Z, Y)
    torch.cuda.synchronize()
    l1.l1dm_free(h)
