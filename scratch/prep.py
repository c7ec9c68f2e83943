import sys, torch, json
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
for name in sys.argv[1:]:
    w = wl.workload(name)
    X = wl.make_points(w, "cuda")
    ts = []
    for rep in range(4):
        torch.cuda.synchronize()
        h = l1.l1dm_prepare(X)
        l1.l1dm_timing_enable(h, True)
        ts.append(l1.l1dm_timing_read(h)['prep_ms'])
        l1.l1dm_free(h)
    print(json.dumps({"w": name, "prep_ms": ts}))
