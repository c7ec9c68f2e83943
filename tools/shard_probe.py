"""One G-way coordinate shard of a workload on one GPU: prepare + Q queries, for an ncu launch
list of the shard's per-query work.  Inputs as bench.py (workloads.py).

    python tools/shard_probe.py --workload c3 --G 8 --queries 10
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15114_b200 as l1  # noqa: E402
from paper_2210_15114_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--G", type=int, default=8)
ap.add_argument("--queries", type=int, default=10)
ap.add_argument("--side-stream", action="store_true", help="queries on a torch side stream, not the default stream")
ap.add_argument("--fresh", action="store_true", help="a different Z per query")
a = ap.parse_args()
w = workloads.workload(a.workload)
X = workloads.make_points(w, device="cuda")
Z = workloads.make_query(w, 0, device="cuda")
n, d = X.shape
kk = (d + a.G - 1) // a.G
Xs = X[:, :kk].contiguous()
h = l1.l1dm_prepare(Xs)
Y = torch.empty(n, Z.shape[1], dtype=torch.float64, device="cuda")
Zs = [workloads.make_query(w, t, device="cuda") for t in range(a.queries)] if a.fresh else [Z]
st = torch.cuda.Stream() if a.side_stream else torch.cuda.current_stream()
torch.cuda.synchronize()
for q in range(a.queries):
    l1.l1dm_matvec(h, Zs[q % len(Zs)], Y, stream=st)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(st)
for q in range(a.queries):
    l1.l1dm_matvec(h, Zs[q % len(Zs)], Y, stream=st)
ev[1].record(st)
torch.cuda.synchronize()
print(f"{a.workload} G={a.G} shard of {kk} coordinates: {ev[0].elapsed_time(ev[1]) / a.queries:.3f} ms per query")
l1.l1dm_free(h)
# per-query times of one more handle's first queries (events around each call)
h = l1.l1dm_prepare(Xs)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.queries + 1)]
evs[0].record(st)
for q in range(a.queries):
    l1.l1dm_matvec(h, Zs[q % len(Zs)], Y, stream=st)
    evs[q + 1].record(st)
torch.cuda.synchronize()
print("per query after a fresh prepare:", " ".join(f"{evs[q].elapsed_time(evs[q + 1]):.2f}" for q in range(a.queries)))
l1.l1dm_free(h)
