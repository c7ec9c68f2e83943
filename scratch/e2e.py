import sys, time, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = wl.workload(name)
Q = 20 if name == "c2" else 5
Xh = wl.make_points(w, "cuda").cpu().pin_memory()
Zh = [wl.make_query(w, t, "cuda").cpu().pin_memory() for t in range(Q if w.fresh_queries else 1)]
Yh = torch.empty((w.n, w.m), dtype=torch.float64).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = l1.l1dm_prepare(Xh); t1 = time.perf_counter()
    for q in range(Q): l1.l1dm_matvec(h, Zh[q % len(Zh)], Yh, block=False)
    t2 = time.perf_counter()
    l1.l1dm_sync(h); t3 = time.perf_counter()
    l1.l1dm_free(h); t4 = time.perf_counter()
    print(f"prep {1e3*(t1-t0):.2f} enqueue {1e3*(t2-t1):.2f} sync {1e3*(t3-t2):.2f} free {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms")
