import sys, torch, numpy as np
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
dev = torch.device("cuda", 0)
out = []
for name in ("c2", "c3", "c5", "c4"):
    w = wl.workload(name)
    X = wl.make_points(w, dev)
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        h = l1.l1dm_prepare(X)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        if it < 3:
            l1.l1dm_free(h)
    ok = True
    if name in ("c2", "c3", "c5") and sys.argv[1] != "nolb":
        sval, perm, rank, hs = l1.l1dm_debug_export(h)
        for k in (0, w.d // 2, w.d - 1):
            col = X[:, k].cpu()
            sv, pi = torch.sort(col, stable=True)
            ok &= np.array_equal(perm[k], pi.numpy().astype(np.uint32)) and np.array_equal(sval[k], sv.numpy())
            ok &= np.array_equal(rank[k][perm[k]], np.arange(w.n, dtype=np.uint32))
    l1.l1dm_free(h)
    del X
    out.append(f"{name} prep ms {min(ts[1:]):.2f} (all {['%.1f' % t for t in ts]}) ok={ok}")
print(sys.argv[1], " | ".join(out), flush=True)
