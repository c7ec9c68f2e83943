import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload("c3")
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
h = l1.l1dm_prepare(X)
Ys = []
for r in range(3):
    Y = l1.l1dm_matvec(h, Z); torch.cuda.synchronize(); Ys.append(Y)
print("c3 scatter bitwise identical across 3 queries:", all(torch.equal(Ys[0], y) for y in Ys[1:]))
print("strategy", l1.l1dm_query_strategy(h, w.m))
