"""Compare query strategies on a workload: python scratch/scat.py c3 gather|scatter|auto [Q]"""
import sys, json, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
import oracle
name, mode = sys.argv[1], sys.argv[2]
Q = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = wl.workload(name)
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
torch.cuda.synchronize()
h = l1.l1dm_prepare(X)
l1.l1dm_set_query_mode(h, mode)
Y = torch.empty((w.n, w.m), dtype=torch.float64, device="cuda")
l1.l1dm_matvec(h, Z, Y); l1.l1dm_sync(h)
l1.l1dm_timing_enable(h, True); l1.l1dm_timing_read(h, reset=True)
for q in range(Q): l1.l1dm_matvec(h, Z, Y)
t = l1.l1dm_timing_read(h); l1.l1dm_sync(h)
l1.l1dm_timing_enable(h, False)
torch.cuda.synchronize(); t0 = time.perf_counter()
for q in range(Q): l1.l1dm_matvec(h, Z, Y)
l1.l1dm_sync(h); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) / Q * 1e3
qms = (t['scan_ms'] + t['accumulate_ms'] + t['colsums_ms']) / Q
rows = np.random.default_rng(0).choice(w.n, 48, replace=False)
Yr = oracle.rows(X.cpu().numpy(), Z.cpu().numpy(), rows)
Yg = Y[torch.as_tensor(rows, device="cuda")].cpu().numpy()
err = max(np.linalg.norm(Yg[:, c] - Yr[:, c]) / np.linalg.norm(Yr[:, c]) for c in range(w.m))
print(json.dumps({"w": name, "mode": mode, "query_ms": round(qms, 3), "wall_ms": round(wall, 3), "scan_ms": round(t['scan_ms'] / Q, 3),
                  "acc_ms": round(t['accumulate_ms'] / Q, 3), "col_ms": round(t['colsums_ms'] / Q, 3),
                  "updates_per_s": w.n * w.d * w.m / (qms * 1e-3), "err": err}))
