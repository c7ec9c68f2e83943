import time, torch
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload("c4"); dev = torch.device("cuda", 0)
X = wl.make_points(w, dev)
Zs = [wl.make_query(w, t, dev) for t in range(10)]
Y = torch.empty((w.n, w.m), dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
for step in range(3):
    t0 = time.perf_counter()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
    e[0].record(s)
    h = l1.l1dm_prepare(X)
    e[1].record(s)
    th = []
    for q in range(10):
        th.append(time.perf_counter())
        l1.l1dm_matvec(h, Zs[q], Y)
        e[q + 2].record(s)
    th.append(time.perf_counter())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    l1.l1dm_free(h)
    t2 = time.perf_counter()
    print("step", step, "prep %.1f" % e[0].elapsed_time(e[1]),
          "q", ["%.1f" % e[i].elapsed_time(e[i + 1]) for i in range(1, 11)],
          "host enqueue ms", ["%.1f" % (1e3 * (th[i + 1] - th[i])) for i in range(10)],
          "wall %.1f free %.1f" % (1e3 * (t1 - t0), 1e3 * (t2 - t1)), flush=True)
