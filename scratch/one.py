"""Run prepare + Q queries of a workload (optionally reduced d) and print per-kernel times."""
import sys, json, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
name = sys.argv[1]; d = int(sys.argv[2]) if len(sys.argv) > 2 else None; Q = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m = int(sys.argv[4]) if len(sys.argv) > 4 else None
w = wl.workload(name, d=d, m=m)
X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
torch.cuda.synchronize()
h = l1.l1dm_prepare(X)
import os
if os.environ.get('WS_GB'): l1.l1dm_set_workspace_limit(h, int(float(os.environ['WS_GB'])*(1<<30)))
Y = torch.empty((w.n, w.m), dtype=torch.float64, device="cuda")
l1.l1dm_matvec(h, Z, Y); torch.cuda.synchronize()
l1.l1dm_timing_enable(h, True); l1.l1dm_timing_read(h, reset=True)
for q in range(Q): l1.l1dm_matvec(h, Z, Y)
t = l1.l1dm_timing_read(h); l1.l1dm_sync(h)
p = l1.l1dm_plan(w.n, w.d, w.m, 126 << 20, 60 << 30)
upd = w.n * w.d * w.m
per = {k: t[k] / max(t[k.replace('_ms', '_launches')], 1) for k in ('scan_ms', 'accumulate_ms', 'colsums_ms')}
qms = (t['scan_ms'] + t['accumulate_ms'] + t['colsums_ms']) / Q
scanB = w.n * w.d * (8 + 12 * w.m); accB = w.n * w.d * (4 + 8 * w.m) + w.n * 8 * w.m
print(json.dumps({"w": name, "n": w.n, "d": w.d, "m": w.m, "prep_ms": round(t['prep_ms'], 2), "query_ms": round(qms, 3),
  "scan_ms_per_query": round(t['scan_ms'] / Q, 3), "acc_ms_per_query": round(t['accumulate_ms'] / Q, 3),
  "scan_GBps": round(scanB / (t['scan_ms'] / Q * 1e-3) / 1e9), "acc_GBps": round(accB / (t['accumulate_ms'] / Q * 1e-3) / 1e9),
  "launches_per_q": t['kernel_launches'] / Q, "plan_kc": p['kc'], "plan_R": p['rows_per_tile'], "mb": p['mb']}))
