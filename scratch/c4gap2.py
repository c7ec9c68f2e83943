import sys, time, torch
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
from paper_2210_15114_b200.distributed import ShardedL1DM
w = wl.workload("c4"); dev = torch.device("cuda", 0)
X = wl.make_points(w, dev)
Zs = [wl.make_query(w, t, dev) for t in range(10)]
Y = torch.empty((w.n, w.m), dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
for variant in sys.argv[1:]:
    for step in range(2):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
        e[0].record(s)
        if "sharded" in variant:
            sh = ShardedL1DM(X, k_range=(0, w.d), stream=s)
            h = sh.handle
        else:
            h = l1.l1dm_prepare(X)
        if "timing" in variant:
            l1.l1dm_timing_enable(h, True)
        e[1].record(s)
        for q in range(10):
            if "sharded" in variant:
                sh.matvec(Zs[q], Y, root=0, overlap_blocks=4)
            else:
                l1.l1dm_matvec(h, Zs[q], Y)
            e[q + 2].record(s)
        tr = l1.l1dm_timing_read(h) if "timing" in variant else {}
        torch.cuda.synchronize()
        if "sharded" in variant: sh.close()
        else: l1.l1dm_free(h)
        print(variant, step, "prep %.1f" % e[0].elapsed_time(e[1]),
              "q", ["%.1f" % e[i].elapsed_time(e[i + 1]) for i in range(1, 11)],
              "kern/q %.1f" % ((tr.get("scan_ms", 0) + tr.get("accumulate_ms", 0) + tr.get("colsums_ms", 0)) / 10), flush=True)
