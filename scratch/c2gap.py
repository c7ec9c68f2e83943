import time, torch
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
from paper_2210_15114_b200.distributed import ShardedL1DM
w = wl.workload("c2"); dev = torch.device("cuda", 0)
X = wl.make_points(w, dev)
Zs = [wl.make_query(w, t, dev) for t in range(20)]
Y = torch.empty((w.n, w.m), dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
for step in range(8):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(23)]
    t = [time.perf_counter()]
    e[0].record(s)
    sh = ShardedL1DM(X, k_range=(0, w.d), stream=s)
    l1.l1dm_timing_enable(sh.handle, True)
    t.append(time.perf_counter())
    e[1].record(s)
    slow = []
    for q in range(20):
        tq = time.perf_counter()
        sh.matvec(Zs[q], Y, root=0, overlap_blocks=4)
        dt = 1e3 * (time.perf_counter() - tq)
        if dt > 0.5: slow.append((q, round(dt, 2)))
        e[q + 2].record(s)
    t.append(time.perf_counter())
    tr = l1.l1dm_timing_read(sh.handle)
    t.append(time.perf_counter())
    sh.close()
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    qs = [e[i].elapsed_time(e[i + 1]) for i in range(1, 21)]
    print("step %d gpu prep %.2f q sum %.2f max %.2f | host prep %.2f enq %.2f read %.2f close %.2f | lib prep %.2f" % (
        step, e[0].elapsed_time(e[1]), sum(qs), max(qs), *[1e3 * (t[i + 1] - t[i]) for i in range(4)], tr["prep_ms"]), slow, flush=True)
