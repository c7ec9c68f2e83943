import sys, time, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload("c2")
X = wl.make_points(w, "cuda"); Zs = [wl.make_query(w, t, "cuda") for t in range(20)]
Y = torch.empty((w.n, 1), dtype=torch.float64, device="cuda")
h = l1.l1dm_prepare(X)
for timing in (False, True):
    l1.l1dm_timing_enable(h, timing)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for q in range(100): l1.l1dm_matvec(h, Zs[q % 20], Y)
        t_host = time.perf_counter() - t0
        e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"timing={timing} host enqueue {t_host/100*1e3:.3f} ms/q, wall {(t1-t0)/100*1e3:.3f} ms/q, gpu {e0.elapsed_time(e1)/100:.3f} ms/q")
    if timing: print(l1.l1dm_timing_read(h))
