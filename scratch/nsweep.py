import torch, sys
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
dev = torch.device("cuda", 0)
for n in [1 << 18, 1 << 19, 3 << 18, 1 << 20, 5 << 18]:
    w = wl.workload("c3", n=n, d=128, m=8)
    X = wl.make_points(w, dev); Z = wl.make_query(w, 0, dev)
    h = l1.l1dm_prepare(X)
    l1.l1dm_timing_enable(h, True)
    for _ in range(3): l1.l1dm_matvec(h, Z)
    torch.cuda.synchronize()
    l1.l1dm_timing_read(h, reset=True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): l1.l1dm_matvec(h, Z)
    b.record(); torch.cuda.synchronize()
    t = l1.l1dm_timing_read(h)
    ms = a.elapsed_time(b) / 10
    acc = t["accumulate_ms"] / max(t["accumulate_launches"], 1)
    print(f"n={n} q={ms:.3f} ms apply={acc:.3f} ms red/s={n*128*8/(acc*1e-3):.3e} strategy={l1.l1dm_query_strategy(h, 8)}", flush=True)
    l1.l1dm_free(h)
