"""Gather vs scatter query time over shapes: python scratch/sweep.py"""
import sys, json, time, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
shapes = [(1 << 20, 128, 64), (1 << 20, 64, 32), (1 << 20, 64, 16), (1 << 20, 64, 8), (1 << 20, 64, 4),
          (1 << 20, 64, 2), (3 << 19, 64, 16), (1 << 21, 64, 16), (1 << 21, 64, 64), (1 << 19, 64, 64),
          (1 << 18, 32, 16), (1 << 16, 32, 64)]
g = torch.Generator(device="cuda"); g.manual_seed(0)
for n, d, m in shapes:
    X = torch.rand((n, d), generator=g, device="cuda") * 2 - 1
    Z = torch.randn((n, m), generator=g, device="cuda")
    Y = torch.empty((n, m), dtype=torch.float64, device="cuda")
    h = l1.l1dm_prepare(X)
    res = {"n": n, "d": d, "m": m, "plan": l1.l1dm_plan(n, d, m)["mb"]}
    ref = None
    for mode in ("gather", "scatter"):
        l1.l1dm_set_query_mode(h, mode)
        l1.l1dm_matvec(h, Z, Y); l1.l1dm_sync(h)
        Q = 5
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(Q): l1.l1dm_matvec(h, Z, Y)
        l1.l1dm_sync(h); e.record(); torch.cuda.synchronize()
        res[mode] = round(s.elapsed_time(e) / Q, 3)
        if ref is None: ref = Y.clone()
        else: res["diff"] = float(((Y - ref).norm(dim=0) / ref.norm(dim=0)).max())
    l1.l1dm_free(h)
    print(json.dumps(res), flush=True)
    del X, Z, Y
