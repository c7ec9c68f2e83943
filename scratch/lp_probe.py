"""Errors and timings of the l_p queries: python scratch/lp_probe.py"""
import sys, json, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2210_15114_b200 as l1, oracle
from conftest import col_rel_l2
rng = np.random.default_rng(0)
for p in (3, 5, 7):
    for n, d, m in [(3000, 4, 17), (20000, 8, 8)]:
        X = rng.standard_normal((n, d)).astype(np.float32); Z = rng.standard_normal((n, m)).astype(np.float32)
        Yr = oracle.brute_lp(X, Z, p) if n <= 3000 else None
        for mode in ("gather", "scatter"):
            h = l1.l1dm_prepare(torch.from_numpy(X).cuda()); l1.l1dm_set_query_mode(h, mode)
            Y = l1.l1dm_matvec_lp(h, p, torch.from_numpy(Z).cuda()).cpu().numpy(); l1.l1dm_free(h)
            if Yr is None:
                rows = np.arange(0, n, 997); e = col_rel_l2(Y[rows], oracle.rows_lp(X, Z, p, rows))
            else:
                e = col_rel_l2(Y, Yr)
            print(json.dumps({"p": p, "n": n, "d": d, "m": m, "mode": mode, "err": e}), flush=True)
from paper_2210_15114_b200 import workloads as wl
for name in ("c3", "c4", "c5"):
    w = wl.workload(name)
    X = wl.make_points(w, "cuda"); Z = wl.make_query(w, 0, "cuda")
    h = l1.l1dm_prepare(X)
    Y = torch.empty((w.n, w.m), dtype=torch.float64, device="cuda")
    for p in (1, 3, 5, 7):
        l1.l1dm_matvec_lp(h, p, Z, Y); l1.l1dm_sync(h)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Q = 3 if name == "c3" else 1
        torch.cuda.synchronize(); s.record()
        for _ in range(Q): l1.l1dm_matvec_lp(h, p, Z, Y)
        e.record(); l1.l1dm_sync(h); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / Q
        print(json.dumps({"w": name, "p": p, "ms": round(ms, 3), "updates_per_s": w.n * w.d * w.m / ms * 1e3,
                          "plan": l1.l1dm_plan(w.n, w.d, w.m)["scatter"]}), flush=True)
    l1.l1dm_free(h); del X, Z, Y; torch.cuda.empty_cache()
