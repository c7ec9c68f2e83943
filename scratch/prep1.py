import sys, torch
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload(sys.argv[1]); dev = torch.device("cuda", 0)
X = wl.make_points(w, dev)
for it in range(2):
    torch.cuda.synchronize()
    h = l1.l1dm_prepare(X); torch.cuda.synchronize(); l1.l1dm_free(h)
