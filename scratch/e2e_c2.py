import time, torch
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
w = wl.workload("c2"); dev = torch.device("cuda", 0)
X = wl.make_points(w, dev); Zs = [wl.make_query(w, t, dev) for t in range(20)]
Xh = X.cpu().pin_memory(); Zh = [z.cpu().pin_memory() for z in Zs]
Yh = torch.empty((w.n, w.m), dtype=torch.float64).pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = l1.l1dm_prepare(Xh)
    t1 = time.perf_counter()
    tq = []
    for q in range(20):
        a = time.perf_counter()
        l1.l1dm_matvec(h, Zh[q], Yh, block=False)
        tq.append(1e3 * (time.perf_counter() - a))
    t2 = time.perf_counter()
    l1.l1dm_sync(h)
    t3 = time.perf_counter()
    l1.l1dm_free(h)
    print(f"prep {1e3*(t1-t0):.1f} ms  enqueue 20q {1e3*(t2-t1):.1f} ms (max {max(tq):.2f})  sync {1e3*(t3-t2):.1f} ms  total {1e3*(t3-t0):.1f}", flush=True)
# the README quick start
X = torch.rand(1 << 20, 128, device="cuda") * 2 - 1
Z = torch.randn(1 << 20, 64, device="cuda")
h = l1.l1dm_prepare(X); Y = l1.l1dm_matvec(h, Z); Y3 = l1.l1dm_matvec_lp(h, 3, Z); l1.l1dm_free(h)
Y2 = l1.l1dm_lpp_even_matvec(X, 2, Z); torch.cuda.synchronize(); print("readme ok", Y.shape, Y3.dtype, Y2.shape)
