#!/usr/bin/env python
"""Benchmark: l1 distance-matrix block product Y = A·Z on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl ours|reference]

One STEP is one pass of the whole hot path over the
workload: prepare (Alg. 1: keys, radix sort, ranks) once, then the workload's
queries (Alg. 2: colsums, gather+scan, rank-gather accumulate; + the NCCL sum of
the partial Y when N > 1).  Default workload c3 (n=2^20, d=128, m=64, prepare once,
100 queries on one fixed Pi; DESIGN.md §7 says why c3).  value = n·d·m·queries /
step time, whole job.  Inputs (1.5 GB prepared state, 256 MB Z) are larger than L2,
so no flush is needed between steps.

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (oracle/, Alg. 1
+ Alg. 2 as written, long double) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_PEAKS_FILE = os.path.join(ROOT, "profiles", "l2_peaks.json")  # tools/l2_probe.cu on a B200
FALLBACK_HBM = 6650.0
PEAK_KIND_RED = ("measured ceiling: max over tools/l2_probe.cu's sweep of fp64 L2 reduction "
                 "patterns (profiles/l2_peaks.json red_ceiling_adds_per_s)")
METRIC = "l1 matvec throughput: n\u00b7d\u00b7m updates/s and achieved HBM GB/s vs peak"  # BASELINE.json


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3",
                    choices=["c1", "c2", "c3", "c4", "c5", "ctx1", "ctx2", "ctx3"])
    ap.add_argument("--queries", type=int, default=None, help="queries per step (default: recipe)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-shard-proxy", action="store_true")
    ap.add_argument("--reduce", default="reduce", choices=["reduce", "allreduce"])
    ap.add_argument("--p", type=int, default=1, choices=[1, 2, 3, 4, 5, 6, 7],
                    help="l_p^p query: odd p sort-based (NEXT-1), even p sort-free (NEXT-4); "
                         "1 = the l1 north star")
    ap.add_argument("--krylov", type=int, default=0,
                    help="K > 0: time block-Krylov top-K singular values of the workload's A "
                         "(NEXT-2) instead of the query loop; block = m/2 fp64 columns")
    ap.add_argument("--l2approx", type=float, default=0.0,
                    help="EPS > 0: approximate l2 product through the l1 engine (NEXT-3): "
                         "embed to k = 12 ln n / EPS^2 coordinates, prepare, run the queries")
    ap.add_argument("--mode", default="auto", choices=["auto", "gather", "scatter"],
                    help="query strategy (include/l1dm.h l1dm_set_query_mode)")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: NCCL per point/column block, or this library's peer-memory sum "
                         "(final pass stores into the owners' inboxes; DESIGN.md §8)")
    ap.add_argument("--no-pattern-probe", action="store_true",
                    help="skip the apply-pattern ceiling probe (tools/apply_probe.cu)")
    ap.add_argument("--overlap-blocks", type=int, default=4,
                    help="N>1: point blocks whose reduce overlaps the remaining accumulate")
    return ap.parse_args()


# --------------------------------------------------------------------------- utils
def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every 5 ms from a
    thread (short timed regions such as c2's ~100 ms still get tens of samples), else
    nvidia-smi every 100 ms."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, [4 reason flags])
        self.proc = None
        self.thread = None
        self.stop_flag = threading.Event()
        self.source = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device's PCI bus id (CUDA and NVML orders can differ)
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), [bool(rs & b) for b in bits]))
                    except Exception:
                        pass
                    self.stop_flag.wait(0.005)

            self.source = "nvml 5 ms"
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.source = "nvidia-smi 100 ms"
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
                try:
                    self.rows.append((float(parts[0]), float(parts[1]),
                                      [parts[2 + j] == "Active" for j in range(4)]))
                except ValueError:
                    pass

    def stop(self):
        self.stop_flag.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        reasons = sorted({self.NAMES[j] for r in self.rows for j in range(4) if r[2][j]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": self.source}


def load_l2_peaks():
    try:
        with open(L2_PEAKS_FILE) as f:
            return json.load(f)
    except Exception:
        return {}


def red_ceiling(l2p):
    """The L2's fp64 reduction ceiling (adds/s): the largest rate any pattern of
    tools/l2_probe.cu's sweep reaches (row widths 32-256 B, buffers 1-64 MiB, localised tables,
    4-16 CTAs per SM); falls back to the earlier single-pattern probe."""
    return float(l2p.get("red_ceiling_adds_per_s", l2p.get("red_row8_adds_per_s", 5.88e11)))


def apply_pattern_probe(n, d):
    """The memory-system ceiling of the scatter apply's own access pattern (tools/apply_probe.cu:
    the perm/sval stream, the Zt row gathers and the 64-bit reductions into Yt, without the scan
    arithmetic or the look-back), compiled and run on this GPU right after the timed region:
    {"best_ms", "median_ms", ...} per launch, or None when nvcc or the probe fails."""
    import subprocess
    import tempfile
    src = os.path.join(ROOT, "tools", "apply_probe.cu")
    try:
        exe = os.path.join(tempfile.gettempdir(), f"l1dm_apply_probe_{os.getpid()}")
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                        src], check=True, capture_output=True, timeout=180)
        out = subprocess.run([exe, str(n), str(d)], check=True, capture_output=True, text=True,
                             timeout=120).stdout
        os.remove(exe)
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        return None


def model_b_bytes(n, d, m):
    """SURVEY §8(d) Model B algorithmic bytes per query: n d (12 + 20 m) + n (12 m + 8)."""
    return n * d * (12 + 20 * m) + n * (12 * m + 8)


def q12_rows(X, count=64, seed=12):
    """SURVEY §8(c) SAMPLE rows (Q12): `count` seeded random rows plus rows 0, n-1, argmin h and
    argmax h (h_i = sum_k x_ik), as row ids on X's device."""
    n = X.shape[0]
    h = X.double().sum(dim=1)
    g = np.random.default_rng(seed)
    r = set(g.integers(0, n, size=count).tolist())
    r |= {0, n - 1, int(torch.argmin(h).item()), int(torch.argmax(h).item())}
    return torch.tensor(sorted(r), dtype=torch.long, device=X.device)


def definition_rows(X, Z, rows, p=1, chunk=1 << 21):
    """y_i = sum_j z_j sum_k |x_ik - x_jk|^p for the listed rows: the definition (
    P:35 for p > 1) in fp64 with plain torch ops on X's device (|R| n d work, no sort, no prefix
    sums): the bench's check of what it timed (the CPU oracle re-checks the same rows at N = 1
    in the cpu_baseline leg)."""
    n = X.shape[0]
    XR = X[rows].double()
    acc = torch.zeros((rows.numel(), Z.shape[1]), dtype=torch.float64, device=X.device)
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        Xc = X[j0:j1].double()
        Zc = Z[j0:j1].double()
        for r in range(rows.numel()):
            D = (Xc - XR[r]).abs_()
            if p != 1:
                D.pow_(p)
            acc[r] += D.sum(dim=1) @ Zc
        del Xc, Zc
    return acc


def col_rel_l2(Y, Yref):
    """Max over columns of ||Y[:,c] - Yref[:,c]||_2 / ||Yref[:,c]||_2 (0/0 = 0, x/0 = inf)."""
    num = torch.linalg.vector_norm((Y - Yref).double(), dim=0)
    den = torch.linalg.vector_norm(Yref.double(), dim=0)
    worst = 0.0
    for a, b in zip(num.tolist(), den.tolist()):
        worst = max(worst, a / b if b > 0 else (0.0 if a == 0 else float("inf")))
    return worst


def sha256_of(t):
    import hashlib
    a = t.detach().cpu().contiguous().numpy()
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()


# --------------------------------------------------------------------------- reference arm
def cpu_oracle_sample(w, queries, budget_dims=None, per_core=True):
    """Time the oracle (as it stands) on a bounded sample: full n, d' coordinates, m' columns."""
    import oracle
    from paper_2210_15114_b200 import workloads as wl
    cores = oracle.num_threads(0)
    n = w.n
    d_s = min(w.d, budget_dims[0] if budget_dims else 32)
    m_s = min(w.m, budget_dims[1] if budget_dims else max(1, min(w.m, cores)))
    ws = wl.workload(w.name, n=n, d=w.d, m=w.m)
    X = wl.make_points(ws, "cpu")[:, :d_s].contiguous().numpy()
    Z = wl.make_query(ws, 0, "cpu")[:, :m_s].contiguous().numpy()
    t0 = time.perf_counter()
    _, order = oracle.alg1(X)
    t_prep = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.alg2(X, order, Z)
    t_q = time.perf_counter() - t0
    upd = n * d_s * m_s
    value = upd * queries / (t_prep + queries * t_q)
    # a single-thread Alg. 2 run gives the per-core rate (2 coordinates, 1 column)
    per_core_rate = None
    if per_core:
        t0 = time.perf_counter()
        oracle.alg2(np.ascontiguousarray(X[:, :2]), np.ascontiguousarray(order[:2]),
                    np.ascontiguousarray(Z[:, :1]), nthreads=1)
        per_core_rate = n * 2 / (time.perf_counter() - t0)
    return {"value": value, "unit": "updates/s", "cores": cores, "kind": "oracle",
            "sample": (f"n={n} (full), d'={d_s} of {w.d} coords, m'={m_s} of {w.m} cols; Alg.1 "
                       f"{t_prep:.2f}s + Alg.2 {t_q:.2f}s per query, step = prep + {queries} "
                       f"queries (query time x{queries})"),
            "per_core_query_updates_per_s": per_core_rate,
            "prep_s": t_prep, "query_s": t_q}


def mix_ceiling(read_fraction):
    """Measured HBM streaming rate (GB/s) at a read fraction of the bytes, piecewise linear
    between the probe's mixes (profiles/hbm_mix.json); None without the probe's file."""
    try:
        h = json.load(open(os.path.join(ROOT, "profiles", "hbm_mix.json")))
        pts = [(0.0, h["write_GBps"]), (1 / 3, h["mix_1r2w_GBps"]), (0.5, h["copy_1r1w_GBps"]),
               (2 / 3, h["mix_2r1w_GBps"]), (1.0, h["read_GBps"])]
    except Exception:
        return None
    x = min(max(read_fraction, 0.0), 1.0)
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        if x <= x1:
            return y0 + (y1 - y0) * (x - x0) / (x1 - x0)
    return pts[-1][1]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2210_15114_b200 import workloads as wl
    w = wl.workload(args.workload)
    Q = args.queries or w.queries
    vals, sample_ms = [], []
    info = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        info = cpu_oracle_sample(w, Q, budget_dims=(64, 16), per_core=(i == 0))
        if i == 0:
            per_core_rate = info["per_core_query_updates_per_s"]
        if i >= args.warmup:
            vals.append(info["value"])
            sample_ms.append((time.perf_counter() - t0) * 1e3)
    value = statistics.mean(vals)
    # ms_per_step is the wall time of the bounded sample each step actually ran (what the
    # driver's clock sees); the full workload's step at this rate is reported beside it
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(sample_ms),
        "full_step_ms_at_this_rate": w.n * w.d * w.m * Q / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (long double accumulation) over f32 inputs", "data": "synthetic",
        "config": {"workload": args.workload, "n": w.n, "d": w.d, "m": w.m, "queries": Q},
        "cpu_baseline": {k: info[k] for k in ("kind", "cores", "sample")}
                        | {"value": value, "unit": "updates/s",
                           "per_core_query_updates_per_s": per_core_rate},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- our arm
def main_ours(args):
    import torch.distributed as dist

    import paper_2210_15114_b200 as l1
    from paper_2210_15114_b200 import workloads as wl
    from paper_2210_15114_b200.distributed import ShardedL1DM, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # test-only overrides (a dry run of the N > 1 path as processes sharing one GPU with gloo:
    # the NCCL-collective path's kernels never wait on each other, so that is safe)
    local = int(os.environ.get("L1DM_BENCH_DEVICE", local))
    backend = os.environ.get("L1DM_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    w = wl.workload(args.workload)
    Q = args.queries or w.queries
    n, d, m = w.n, w.d, w.m
    stream = torch.cuda.current_stream(dev)

    # inputs resident in HBM before timing: full X regenerated per rank from the seed
    Xfull = wl.make_points(w, dev)
    x_sha = sha256_of(Xfull) if rank == 0 else None
    k0, k1 = shard_range(d, rank, world)
    X = Xfull[:, k0:k1].contiguous() if world > 1 else Xfull
    del Xfull
    torch.cuda.empty_cache()
    if w.fresh_queries:
        Zs = [wl.make_query(w, t, dev) for t in range(Q)]
    else:
        Zs = [wl.make_query(w, 0, dev)]
    z_sha = None
    if rank == 0:
        import hashlib
        hz = hashlib.sha256()
        for z in Zs:
            hz.update(sha256_of(z).encode())
        z_sha = hz.hexdigest() if len(Zs) > 1 else sha256_of(Zs[0])
    Y = torch.empty((n, m), dtype=torch.float64, device=dev)
    kr = (0, k1 - k0)

    peer = {}  # collective="peer": the symmetric buffers are set up once, reused every step

    def one_step(timing=False, qev=None):
        if args.collective == "peer" and world > 1 and not peer:
            from paper_2210_15114_b200.distributed import PeerGroup
            peer["g"] = PeerGroup(n, m, result_ranks=(tuple(range(world))
                                                      if args.reduce == "allreduce" else (0,)))
        sh = ShardedL1DM(X, k_range=kr, stream=stream, mode=args.mode, p=args.p,
                         peer_group=peer.get("g"))
        sh.world = world
        if timing and sh.handle is not None and args.p % 2 == 1:
            l1.l1dm_timing_enable(sh.handle, True)
        for q in range(Q):
            if qev is not None:
                qev[2 * q].record(stream)
            sh.matvec(Zs[q % len(Zs)], Y, root=None if args.reduce == "allreduce" else 0,
                      overlap_blocks=args.overlap_blocks, collective=args.collective)
            if qev is not None:
                qev[2 * q + 1].record(stream)
        return sh

    for _ in range(args.warmup):
        sh = one_step()
        torch.cuda.synchronize()
        sh.close()
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    timings = []
    strategy = None
    hl0 = l1.l1dm_handleless_launches()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    ev0.record(stream)
    # per-query events in the last timed step (median / spread of the query time)
    qev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * Q)]
    torch.cuda.nvtx.range_push(f"bench {args.workload}: {args.steps} timed steps")
    for s in range(args.steps):
        last = s == args.steps - 1
        step_ev[2 * s].record(stream)
        torch.cuda.nvtx.range_push(f"step {s}")
        sh = one_step(timing=True, qev=qev if last else None)
        torch.cuda.nvtx.range_pop()
        step_ev[2 * s + 1].record(stream)
        if sh.handle is not None and args.p % 2 == 1:
            timings.append(l1.l1dm_timing_read(sh.handle))  # syncs the stream (host only)
        if sh.handle is not None and args.p % 2 == 1:
            strategy = l1.l1dm_query_strategy(sh.handle, m)  # (runs serves every odd p)
        if not last:
            sh.close()  # the last step's handle is validated after the timed region
    torch.cuda.nvtx.range_pop()
    ev1.record(stream)
    hl_launches = l1.l1dm_handleless_launches() - hl0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    ms_total = ev0.elapsed_time(ev1)
    step_ms = [step_ev[2 * s].elapsed_time(step_ev[2 * s + 1]) for s in range(args.steps)]
    q_ms = [qev[2 * q].elapsed_time(qev[2 * q + 1]) for q in range(Q)]

    # ---- what was timed, validated (queries 0 and Q-1): Y still
    # holds query Q-1 of the last timed step; query 0 is re-run on the same handle (same
    # strategy, recycled workspace).  Checked on SURVEY's rows against the definition in fp64.
    root_has_y = rank == 0
    Ylast = Y.clone() if root_has_y else None
    sh.matvec(Zs[0], Y, root=None if args.reduce == "allreduce" else 0,
              overlap_blocks=args.overlap_blocks, collective=args.collective)
    torch.cuda.synchronize()
    sh.close()
    parity = parity_inputs = None
    if root_has_y:
        Xv = wl.make_points(w, dev)          # the full X (every rank holds only its shard)
        rows = q12_rows(Xv)
        checks = []
        for label, Yq, Zq in ((f"query {Q - 1} (last timed)", Ylast, Zs[(Q - 1) % len(Zs)]),
                              ("query 0 (re-run on the timed handle)", Y, Zs[0])):
            want = definition_rows(Xv, Zq, rows, p=args.p)
            got = Yq[rows]
            checks.append({"query": label, "max_col_rel_l2": col_rel_l2(got, want),
                           "bit_exact": bool(torch.equal(got, want))})
        exact_required = w.x_dist == "int256" and w.z_dist == "pm1"  # c5: integers < 2^53
        worst = max(c["max_col_rel_l2"] for c in checks)
        parity = {"rows": int(rows.numel()),
                  "row_set": "64 seeded random + {0, n-1, argmin h, argmax h} (SURVEY Q12)",
                  "reference": "definition P:149/P:171 in fp64 on the device (torch, |R| n d)",
                  "queries": checks, "max_col_rel_l2": worst, "tolerance": 1e-9,
                  "exact_required": exact_required,
                  "pass": (all(c["bit_exact"] for c in checks) if exact_required
                           else worst <= 1e-9)}
        parity_inputs = (Xv, rows, [(Ylast, Zs[(Q - 1) % len(Zs)]), (Y, Zs[0])])
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    upd_step = n * d * m * Q
    value = upd_step / (ms_step * 1e-3)

    # per-kernel device times (CUDA events on the library's stream), this rank
    agg = {k: sum(tt[k] for tt in timings) for k in timings[0]} if timings else {}
    prep_ms = statistics.mean(tt["prep_ms"] for tt in timings) if timings else None
    nq = max(agg.get("queries", 0), 1)
    query_kernel_ms = ((agg["colsums_ms"] + agg["scan_ms"] + agg["accumulate_ms"]) / nq
                       if agg else None)
    hbm_peak, peak_kind = load_peaks()
    dl = k1 - k0
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    plan = l1.l1dm_plan(n, max(dl, 1), m, l2_bytes, 0, mode=args.mode)
    qb = model_b_bytes(n, dl, m)
    kern = {
        "scan": {"ms_total": agg.get("scan_ms"), "launches": agg.get("scan_launches")},
        "accumulate": {"ms_total": agg.get("accumulate_ms"),
                       "launches": agg.get("accumulate_launches")},
    }
    for kv in kern.values():
        kv["ms_per_launch"] = kv["ms_total"] / max(kv["launches"] or 1, 1) if kv["ms_total"] else None
    l2p = load_l2_peaks()
    if args.p % 2 == 0:
        # even p (NEXT-4, sort-free): two fp64 contractions on DMMA (moment reduce + expand);
        # bound: the fp64 tensor rate measured by tools/fp64_probe.cu (fallback: derived from
        # the unit count, 64 fp64 FMA/clk/SM x 148 SMs x 2 flops x the max SM clock)
        for kv in kern.values():
            kv["achieved_GBps"] = None
        # the contractions the method needs: W_t = (X^t)^T Z for t = 1..p-1 and the expansion
        # sum_t X^(p-t) W_t, 2 n d m flops each per power (S, G and hp are O(n (d + m)))
        flops = 4.0 * n * dl * m * (args.p - 1)
        ach = flops / (ms_step * 1e-3 / Q) / 1e12
        try:
            fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
            peak, pk = float(fp["dmma_m8n8k4_tflops"]), "measured (tools/fp64_probe.cu)"
        except Exception:
            peak, pk = 64 * 148 * 2 * 1.965e9 / 1e12, "derived: 64 fp64 FMA/clk/SM x 148 x 1.965 GHz"
        dominant = "query"
        roof = {"bound": "tensor", "kernel": "whole query (k12 reduce + k13 fold + k14 expand)",
                "achieved": ach, "peak": peak, "unit": "TFLOP/s (fp64 DMMA)", "peak_kind": pk,
                "frac": ach / peak, "alg_flops_per_query": flops}
    elif strategy == "runs":
        # runs mode (tie-heavy data): "scan" = the run histogram (one fp64 L2
        # reduction per update into the L2-resident (coordinate, run, column) table, run ids
        # and Z rows streamed in point order) + the prefix over runs; "accumulate" = the
        # expansion (per pair a run id from HBM and a U row from the L2-resident table).  HBM
        # moves only 2 n d (run ids) + n m (4 + 8) bytes per query, so the histogram's
        # reductions bound the query: roofline in reductions/s against the measured probe.
        red = agg.get("queries", 0) * n * dl * m
        sc = kern["scan"]
        kern["scan"]["alg_reductions"] = red
        hbm_q = 2 * n * dl + n * m * 12 + n * 8
        for kv in kern.values():
            kv["achieved_GBps"] = None
        dominant = "scan"
        ach = (red / (sc["ms_total"] * 1e-3) / 1e9) if sc["ms_total"] else None
        peak = red_ceiling(l2p) / 1e9
        roof = {"bound": "l2_fp64_reductions",
                "note": "the histogram's reductions concentrate on a 3 MiB table (dl x 256 x m); "
                        "peak = the ceiling of tools/l2_probe.cu's sweep (the best of every "
                        "pattern, including 3 MiB buffers and localised tables)",
                "kernel": "run histogram (k20_runs_hist + the scan over runs)",
                "achieved": ach, "peak": peak, "unit": "G fp64 reductions/s",
                "peak_kind": PEAK_KIND_RED,
                "frac": (ach / peak) if ach else None,
                "alg_reductions_per_launch": red / max(sc["launches"] or 1, 1),
                "hbm_bytes_per_query": hbm_q,
                "hbm_GBps": (hbm_q / (query_kernel_ms * 1e-3) / 1e9) if query_kernel_ms else None}
    elif args.p > 1:
        # l_p^p, odd p: the seq scan with p+1 moments in both strategies.
        # scatter: the apply pass's fp64 L2 reductions, one per update, as for p = 1.
        # gather: HBM bytes per query = per (i,k): two passes of perm/sval (16) and Zt rows
        # (8m) gathered from HBM, the U store (8m) and k6's rank + U gather (4 + 8m); Y 8m per
        # point.  Reported against the HBM peak for the whole query (its kernels interleave).
        for kv in kern.values():
            kv["achieved_GBps"] = None
        if plan["scatter"]:
            red = agg.get("queries", 0) * n * dl * m
            acc = kern["accumulate"]
            dominant = "accumulate"
            ach = (red / (acc["ms_total"] * 1e-3) / 1e9) if acc["ms_total"] else None
            peak = red_ceiling(l2p) / 1e9
            roof = {"bound": "l2_fp64_reductions", "kernel": f"apply (k5_scan_seq<mb,APPLY,{args.p}>)",
                    "achieved": ach, "peak": peak, "unit": "G fp64 reductions/s",
                    "peak_kind": PEAK_KIND_RED,
                    "frac": (ach / peak) if ach else None}
        else:
            qbytes = n * dl * (16 + 8 * m + 8 * m + 4 + 8 * m) + n * 8 * m
            ach = qbytes / (query_kernel_ms * 1e-3) / 1e9 if query_kernel_ms else None
            dominant = "query"
            roof = {"bound": "hbm", "kernel": "whole query (seq reduce/apply-store + k6)",
                    "achieved": ach, "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                    "frac": (ach / hbm_peak) if ach else None, "alg_bytes_per_query": qbytes}
    elif plan["scatter"] and m > 1:
        # scatter mode: per column block, "accumulate" = the apply (perm/sval
        # streamed from HBM, one Zt row gathered from L2 per pair, one 8-byte L2 reduction per
        # update; by default single-pass, its tile prefixes by look-back), "scan" = the two-pass
        # form's reduce + prefix (L1DM_SCATTER_LB=0 only).  The apply pass is bounded by the L2's
        # reduction throughput: roofline in reductions/s against the measured probe.
        mb = plan["mb"]
        kern["scan"]["alg_bytes"] = agg.get("scan_pairs", 0) * (8 + 4 * mb)
        kern["accumulate"]["alg_reductions"] = agg.get("queries", 0) * n * dl * m
        kern["accumulate"]["alg_bytes"] = agg.get("accumulate_pairs", 0) * (8 + 4 * mb) + \
            kern["accumulate"]["alg_reductions"] * 8
        for kv in kern.values():
            kv["achieved_GBps"] = (kv["alg_bytes"] / (kv["ms_total"] * 1e-3) / 1e9
                                   if kv["ms_total"] else None)
        acc = kern["accumulate"]
        dominant = "accumulate"
        ach = (acc["alg_reductions"] / (acc["ms_total"] * 1e-3) / 1e9) if acc["ms_total"] else None
        peak = red_ceiling(l2p) / 1e9
        single = not kern["scan"]["launches"]  # the default single-pass apply (k5_scan_lb)
        roof = {"bound": "l2_fp64_reductions",
                "kernel": ("apply (k5_scan_lb<mb>: look-back prefixes + 64-bit L2 reductions)"
                           if single else "apply (k5_scan_seq<mb,APPLY>)"),
                "achieved": ach, "peak": peak,
                "peak_kind": PEAK_KIND_RED if l2p else "fallback (earlier probe)",
                "unit": "G fp64 reductions/s", "frac": (ach / peak) if ach else None,
                "alg_reductions_per_launch": acc["alg_reductions"] / max(acc["launches"] or 1, 1)}
    else:
        # gather mode: algorithmic bytes (SURVEY §8(d) Model B, split by kernel)
        #   scan       per (point, coordinate): perm 4 + sval 4 + Z row 4m + U row 8m
        #   accumulate per (point, coordinate): rank 4 + U row 8m; per point and query: Y 8m + h 8
        kern["scan"]["alg_bytes"] = agg.get("scan_pairs", 0) * (8 + 12 * m)
        kern["accumulate"]["alg_bytes"] = (agg.get("accumulate_pairs", 0) * (4 + 8 * m) +
                                           agg.get("queries", 0) * n * (8 * m + 8))
        for kv in kern.values():
            kv["achieved_GBps"] = (kv["alg_bytes"] / (kv["ms_total"] * 1e-3) / 1e9
                                   if kv["ms_total"] else None)
        dominant = max(kern, key=lambda k: kern[k]["ms_total"] or 0.0)
        ach = kern[dominant]["achieved_GBps"]
        roof = {"bound": "hbm", "kernel": dominant, "achieved": ach, "peak": hbm_peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": (ach / hbm_peak) if ach else None,
                "alg_bytes_per_launch": (kern[dominant]["alg_bytes"] /
                                         max(kern[dominant]["launches"] or 1, 1)),
                "frac_of_8TBps": (ach / 8000.0) if ach else None}
        # HBM rate depends on the read:write mix (tools/hbm_mix_probe.cu -> profiles/hbm_mix.json:
        # 1 read : 2 writes streams at ~4.9 TB/s, reads alone at ~7.1); the scan reads
        # 8 + 4m and writes 8m bytes per pair, the accumulate almost only reads
        rfrac = {"scan": (8 + 4 * m) / (8 + 12 * m),
                 "accumulate": (4 + 8 * m) / (4 + 8 * m + 16.0 * m / max(dl, 1))}[dominant]
        mixc = mix_ceiling(rfrac)
        if mixc and ach:
            roof["mix_ceiling_GBps"] = mixc
            roof["frac_of_mix_ceiling"] = ach / mixc
            roof["read_fraction"] = rfrac
        if plan["scatter"]:
            # m == 1 scatter mode: z (4 MB) and Y (8 MB) live in L2; per (point, coordinate) the
            # query makes two random 32-byte sector accesses (the z gather of the reduce pass and
            # the fp64 reduction into Y of the apply pass) — bound by the L2's random-sector
            # rate, measured by tools/l2_probe.cu (profiles/l2_peaks.json gather_sector_GBps)
            # per (point, coordinate): one random 4-byte z gather (reduce pass) and one random
            # fp64 reduction into Y (apply pass), each at the L2's measured per-lane rate
            # (tools/l2_probe.cu: gather_lane_per_s, red_lane_per_s); the passes run in turn,
            # so the ceiling is the harmonic combination of the two rates
            single = not kern["scan"]["launches"]  # default: the single-pass apply (k5_scan_lb<1>)
            sc = kern["accumulate"] if single else kern["scan"]
            pairs = agg.get("accumulate_pairs" if single else "scan_pairs", 0)
            g = max(l2p.get("gather_lane_per_s", 2.69e11), l2p.get("gather_lane_4MiB_per_s", 0))
            r = max(l2p.get("red_lane_per_s", 1.745e11), l2p.get("red_lane_8MiB_per_s", 0))
            peak = 1.0 / (1.0 / g + 1.0 / r) / 1e9
            ach = pairs / (sc["ms_total"] * 1e-3) / 1e9 if sc["ms_total"] else None
            roof = {"bound": "l2_random_access",
                    "kernel": ("apply (k5_scan_lb<1>: gather, look-back, 64-bit reductions)" if single
                               else "scan (k5_scan_m1 reduce/prefix/apply)"),
                    "achieved": ach, "peak": peak,
                    "unit": "G (point, coordinate) pairs/s: one random 4-B gather + one random "
                            "fp64 reduction each",
                    "peak_kind": "measured (tools/l2_probe.cu single-lane gather and reduction "
                                 "rates, harmonic combination)",
                    "frac": (ach / peak) if ach else None,
                    "note": "m = 1: L2-resident z and Y; HBM carries only the sorted tables"}
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.workload}.json")
    if os.path.exists(prof) and args.p == 1:
        try:
            tr = json.load(open(prof))
            strat = strategy or ("scatter" if plan["scatter"] else "gather")
            traffic = tr.get(f"{strat}_{dominant}", tr.get(dominant))
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    # the HBM view of the same kernel (MEASURED_PEAKS.json): its ncu DRAM bytes per launch over
    # its event-timed launch duration, against the copy peak
    dk = kern.get(dominant) if isinstance(kern.get(dominant), dict) else None
    if traffic and dk and dk.get("ms_per_launch"):
        roof["dram_GBps"] = traffic / (dk["ms_per_launch"] * 1e-3) / 1e9
        roof["dram_frac_of_hbm_peak"] = roof["dram_GBps"] / hbm_peak
    # the apply's own access pattern without its arithmetic (tools/apply_probe.cu), on this GPU
    # after the timed region: the fraction of that pattern's ceiling the kernel reaches
    if (plan and plan.get("scatter") and m > 1 and plan.get("mb") == 8 and args.p == 1
            and dominant == "accumulate" and not kern["scan"]["launches"] and world == 1
            and not args.no_pattern_probe):
        pr = apply_pattern_probe(n, dl)
        acc_ms = kern["accumulate"].get("ms_per_launch")
        if pr and acc_ms and pr.get("n") == n:
            roof["pattern_ceiling"] = {
                "ms_per_launch_best": pr["apply_pattern_ms"],
                "ms_per_launch_median": pr["apply_pattern_median_ms"],
                "frac_of_best": pr["apply_pattern_ms"] / acc_ms,
                "frac_of_median": pr["apply_pattern_median_ms"] / acc_ms,
                "how": "tools/apply_probe.cu: the apply's perm/sval stream, Zt row gathers and "
                       "64-bit L2 reductions (same tiles, grid and L2 hints) without the scan "
                       "arithmetic or the look-back; best, and median of the last 32 of 800 "
                       "back-to-back launches with their clears (sustained, as in a step)"}
    # the U-materialising design's HBM floor (Model B bytes) over the measured query time:
    # above 1.0 means the query beats that design's roofline
    roof["model_b_hbm_equivalent_frac"] = (qb / (query_kernel_ms * 1e-3) / 1e9 / hbm_peak
                                           if query_kernel_ms and args.p % 2 == 1 else None)
    result = {
        "metric": METRIC,
        "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "input_dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "n": n, "d": d, "m": m, "queries_per_step": Q,
                   "fresh_queries": w.fresh_queries, "parallelism": f"coord-shard x{world}",
                   "collective": (f"{args.reduce} over {args.collective}" if world > 1 else None),
                   "overlap_blocks": (args.overlap_blocks if world > 1 else None),
                   "mode": args.mode,
                   "strategy": strategy or ("scatter" if plan["scatter"] else "gather"),
                   "query": "l1" if args.p == 1 else f"lp^p, p={args.p}",
                   "columns_per_block": plan["mb"],
                   "l2": "inputs > L2 (prepared state 12*n*d B), no flush"},
        "gpu_launches": int(agg.get("kernel_launches", 0)) + hl_launches,
        "prepare_ms": prep_ms,
        # prepare as keys/s and GB/s against the 16-B compulsory and 76-B pass
        # models (per key: X read + sval/perm/rank write; keys, histogram, 4 radix passes, ranks)
        "prepare": ({"keys_per_s": n * dl / (prep_ms * 1e-3),
                     "GBps_16B_model": 16.0 * n * dl / (prep_ms * 1e-3) / 1e9,
                     "GBps_76B_model": 76.0 * n * dl / (prep_ms * 1e-3) / 1e9,
                     "frac_76B_of_hbm_peak": 76.0 * n * dl / (prep_ms * 1e-3) / 1e9 / hbm_peak}
                    if prep_ms else None),
        "step_ms_each": step_ms,
        "ms_per_step_median": statistics.median(step_ms),
        "query_ms": (ms_step - (prep_ms or 0.0)) / Q,
        "query_ms_last_step": {"median": statistics.median(q_ms), "min": min(q_ms),
                               "max": max(q_ms), "mean": statistics.mean(q_ms)},
        "inputs_sha256": {"X": x_sha, "Z": z_sha},
        "parity": parity,
        "query_kernel_ms": query_kernel_ms,
        "kernels": kern,
        "colsums_ms_per_launch": (agg["colsums_ms"] / max(agg["colsums_launches"], 1)
                                  if agg else None),
        "model_b_GBps_per_query": qb / (query_kernel_ms * 1e-3) / 1e9 if query_kernel_ms else None,
        "roofline": roof,
        "clocks": clk,
    }
    # ---- multi-GPU readiness on one GPU (compute only): one step of a G = 8 coordinate shard
    # (ceil(d/8) coordinates: prepare + the same queries) against the full step; t1 / (G t_G)
    # is the efficiency an 8-GPU run could reach before any collective cost
    if world == 1 and args.p % 2 == 1 and d >= 8 and not args.no_shard_proxy:
        G = 8
        kk = -(-d // G)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c_ = torch.cuda.Event(enable_timing=True)
        Ys = torch.empty_like(Y)  # Y still holds the validated query-0 rows
        Xs = X[:, :kk].contiguous()  # what a rank holds at N > 1 (its slice, made contiguous)

        def shard_step(colblocks):
            """prepare + Q queries on the shard; colblocks: the call each rank makes at N > 1
            (scatter strategy, --overlap-blocks > 1: column-block-major output, one event per
            block for the per-block reduce) instead of the row-major l1dm_matvec"""
            times = None
            for _ in range(2):  # one untimed, one timed
                torch.cuda.synchronize()
                a.record(stream)
                hs = l1.l1dm_prepare(Xs, stream=stream)
                c_.record(stream)
                l1.l1dm_set_query_mode(hs, args.mode)
                if colblocks:
                    sc_, mb_, ncb_ = l1.binding.l1dm_query_layout(hs, m)
                    if not (sc_ and m > 1):
                        l1.l1dm_free(hs)
                        return None
                    Yb = torch.empty((ncb_, n, mb_), dtype=torch.float64, device=dev)
                    evs = [torch.cuda.Event() for _ in range(ncb_)]
                for q in range(Q):
                    if colblocks:
                        l1.binding.l1dm_matvec_colblocks(hs, Zs[q % len(Zs)], Yb, evs, stream=stream)
                    elif args.p == 1:
                        l1.l1dm_matvec(hs, Zs[q % len(Zs)], Ys, stream=stream)
                    else:
                        l1.l1dm_matvec_lp(hs, args.p, Zs[q % len(Zs)], Ys, stream=stream)
                b.record(stream)
                torch.cuda.synchronize()
                l1.l1dm_free(hs)
                times = (a.elapsed_time(b), a.elapsed_time(c_))
            return times

        t_shard, t_shard_prep = shard_step(False)
        cb_times = shard_step(True) if args.p == 1 and args.overlap_blocks > 1 else None
        del Ys, Xs
        result["shard_proxy"] = {
            "G": G, "coords_per_shard": kk, "t1_ms_per_step": ms_step,
            "t_shard_ms_per_step": t_shard, "compute_efficiency": ms_step / (G * t_shard),
            "t1_prepare_ms": prep_ms, "t_shard_prepare_ms": t_shard_prep,
            "t1_query_ms": (ms_step - (prep_ms or 0.0)) / Q,
            "t_shard_query_ms": (t_shard - t_shard_prep) / Q,
            "note": "one B200: a step (prepare + the same queries) on coordinates [0, ceil(d/8)) "
                    "vs the full step; excludes the cross-GPU sum (DESIGN.md §8)"}
        if cb_times:
            # what each rank computes at N > 1 in the scatter strategy (bench.py --gpus N runs
            # ShardedL1DM.matvec with --overlap-blocks 4: l1dm_matvec_colblocks, then the
            # per-block reduce and the root's l1dm_unblock, both part of the collective phase)
            result["shard_proxy"].update({
                "t_shard_colblocks_ms_per_step": cb_times[0],
                "t_shard_colblocks_query_ms": (cb_times[0] - cb_times[1]) / Q,
                "compute_efficiency_colblocks": ms_step / (G * cb_times[0]),
                "note_colblocks": "per-rank call of the N > 1 scatter path (column-block-major "
                                  "output for the per-block reduce)"})
    # ---- e2e through the public API with HOST buffers (pinned), N=1 only
    if world == 1 and not args.no_e2e:
        Xh = X.cpu().pin_memory()
        Zh = [z.cpu().pin_memory() for z in Zs]
        Yh = torch.empty((n, m), dtype=torch.float64).pin_memory()

        def e2e_step():
            if args.p % 2 == 0:
                for q in range(Q):
                    l1.l1dm_lpp_even_matvec(Xh, args.p, Zh[q % len(Zh)], Yh)
            else:
                h = l1.l1dm_prepare(Xh)
                l1.l1dm_set_query_mode(h, args.mode)
                for q in range(Q):  # pinned buffers: copies of query q+1 / q-1 overlap query q
                    if args.p == 1:
                        l1.l1dm_matvec(h, Zh[q % len(Zh)], Yh, block=False)
                    else:
                        l1.l1dm_matvec_lp(h, args.p, Zh[q % len(Zh)], Yh, block=False)
                l1.l1dm_sync(h)
                l1.l1dm_free(h)

        # one untimed step first (first-touch costs of the pinned staging path), then the same
        # number of timed steps as the device-timed measurement, wall clock
        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / args.steps
        result["e2e"] = {"value": upd_step / e2e_s, "unit": "updates/s",
                         "h2d_bytes_per_step": int(Xh.numel() * 4 * (Q if args.p % 2 == 0 else 1)
                                                   + Q * n * m * 4),
                         "d2h_bytes_per_step": int(Q * n * m * 8),
                         "note": "per step: l1dm_prepare(pinned host X) + per query "
                                 "l1dm_matvec(pinned host Z, pinned host Y), copies overlapped "
                                 "across queries, one l1dm_sync at the end (inside the timed "
                                 "region); 1 untimed step, then mean over --steps steps"}
        del Xh, Zh, Yh
    if world > 1:
        # SURVEY §8(d) multi-GPU protocol: the per-query compute without the collective, and
        # the collective alone at the same message size (bus bandwidth), device-timed, max over
        # ranks
        sh = ShardedL1DM(X, k_range=kr, stream=stream, mode=args.mode, p=args.p)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nq = min(Q, 5)
        dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for q in range(nq):
            sh.partial(Zs[q % len(Zs)], Y)
        b.record(stream)
        torch.cuda.synchronize()
        comp = a.elapsed_time(b) / nq
        sh.close()
        dist.barrier()
        a.record(stream)
        for _ in range(nq):
            if args.reduce == "allreduce":
                dist.all_reduce(Y, op=dist.ReduceOp.SUM)
            else:
                dist.reduce(Y, dst=0, op=dist.ReduceOp.SUM)
        b.record(stream)
        torch.cuda.synchronize()
        coll = a.elapsed_time(b) / nq
        tt = torch.tensor([comp, coll], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        comp, coll = (float(v) for v in tt.tolist())
        msg = n * m * 8
        factor = 2.0 * (world - 1) / world if args.reduce == "allreduce" else (world - 1) / world
        result["multi_gpu"] = {
            "compute_only_ms_per_query": comp, "collective_alone_ms": coll,
            "message_bytes": msg, "collective": args.reduce,
            "bus_GBps": factor * msg / (coll * 1e-3) / 1e9 if coll > 0 else None,
            "note": "partial A^(K_g) Z per rank (no collective) and the collective alone on an "
                    "n x m fp64 buffer; device-timed, max over ranks; NCCL bus-bandwidth factor"}
    if world > 1 and not args.no_e2e:
        # N > 1: every rank uploads its coordinate shard of X and each query's Z from pinned
        # host memory, the sharded query + collective runs as in the timed step, and the root
        # reads every Y back into pinned host memory; wall time, max over ranks
        Xh = X.cpu().pin_memory()
        Zh = [z.cpu().pin_memory() for z in Zs]
        Yh = torch.empty((n, m), dtype=torch.float64).pin_memory() if rank == 0 else None
        Zd = torch.empty((n, m), dtype=torch.float32, device=dev)
        root = None if args.reduce == "allreduce" else 0

        def e2e_step():
            Xd = Xh.to(dev, non_blocking=True)
            sh = ShardedL1DM(Xd, k_range=kr, stream=stream, mode=args.mode, p=args.p,
                             peer_group=peer.get("g"))
            for q in range(Q):
                Zd.copy_(Zh[q % len(Zh)], non_blocking=True)
                sh.matvec(Zd, Y, root=root, overlap_blocks=args.overlap_blocks,
                          collective=args.collective)
                if rank == 0:
                    Yh.copy_(Y, non_blocking=True)
            torch.cuda.synchronize()
            sh.close()

        e2e_step()  # untimed: first-touch costs
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64,
                          device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_s = float(dt.item())
        result["e2e"] = {"value": upd_step / e2e_s, "unit": "updates/s",
                         "h2d_bytes_per_step": int(n * d * 4 + world * Q * n * m * 4),
                         "d2h_bytes_per_step": int(Q * n * m * 8),
                         "note": "per rank: pinned host X shard + each query's Z uploaded, "
                                 "sharded query + collective, root reads Y into pinned host "
                                 "memory; 1 untimed step, then the mean over --steps steps, "
                                 "wall time, max over ranks"}
        del Xh, Zh, Yh, Zd
    # ---- CPU baseline: the oracle on the host cores, bounded sample, rank 0 at N=1; the same
    # leg re-checks the validated rows with the oracle itself (the definition, in C, long double)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_oracle_sample(w, Q, budget_dims=(64, 16))
            result["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind",
                                                         "sample", "per_core_query_updates_per_s")}
            if w.n <= 4096:  # c1 also times BRUTE, O(n^2 (d + m))
                import oracle
                Xb, Zb = X.cpu().numpy(), Zs[0].cpu().numpy()
                t0 = time.perf_counter()
                oracle.brute(Xb, Zb)
                result["cpu_baseline"]["brute_s_per_query"] = time.perf_counter() - t0
        except Exception as e:  # the baseline is reported, never required
            result["cpu_baseline"] = {"value": None, "error": str(e)}
        if parity is not None and args.p % 2 == 1:
            import oracle
            Xv, rows, pairs = parity_inputs
            Xh, rh = Xv.cpu().numpy(), rows.cpu().numpy()
            Zcat = np.concatenate([zq.cpu().numpy() for _, zq in pairs], axis=1)
            t0 = time.perf_counter()
            Yr = (oracle.rows(Xh, Zcat, rh) if args.p == 1 else oracle.rows_lp(Xh, Zcat, args.p, rh))
            worst_o, exact_o = 0.0, True
            for i, (yq, _) in enumerate(pairs):
                want = torch.from_numpy(np.ascontiguousarray(Yr[:, i * m:(i + 1) * m])).to(dev)
                got = yq[rows]
                worst_o = max(worst_o, col_rel_l2(got, want))
                exact_o = exact_o and bool(torch.equal(got, want))
            parity["oracle"] = {"max_col_rel_l2": worst_o, "bit_exact": exact_o,
                                "seconds": time.perf_counter() - t0,
                                "reference": "oracle.rows (C, long double): the same rows"}
            parity["pass"] = parity["pass"] and (exact_o if parity["exact_required"]
                                                 else worst_o <= 1e-9)
    parity_inputs = None
    if w.name in wl.PAPER_TABLE3:  # context only (SURVEY §8(d) ctx): the paper's M1/Numba times
        pp, pq = wl.PAPER_TABLE3[w.name]
        result["paper_context"] = {
            "paper_prepare_s": pp, "paper_avg_query_s": pq,
            "paper_hardware": "2021 M1 MacBook Pro, Python 3.9 + NumPy/Numba (P:360)",
            "this_prepare_s": (prep_ms or 0.0) * 1e-3, "this_avg_query_s": result["query_ms"] * 1e-3,
            "data": "synthetic stand-in of the same shape (Table 3, P:336-345)"}
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0 and parity is not None and not parity["pass"]:
        print(f"bench: PARITY FAILED on the timed work: {json.dumps(parity)}", file=sys.stderr)
        return 1
    return 0


def main_krylov(args):
    """NEXT-2 measurement: prepare once, then block Krylov for the top-K singular values, every
    step in the library (products, fp64 DMMA Gram-Schmidt, Jacobi; 1 GPU).  value = updates/s
    over the products (n d columns)."""
    import paper_2210_15114_b200 as l1
    from paper_2210_15114_b200 import workloads as wl
    from paper_2210_15114_b200.binding import Operator
    from paper_2210_15114_b200.krylov import block_krylov, fp64_product
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = wl.workload(args.workload)
    n, d, m = w.n, w.d, w.m
    X = wl.make_points(w, dev)
    b = max(1, min(96, m // 2))
    k = min(args.krylov, b)
    times, infos = [], []
    for step in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h = l1.l1dm_prepare(X)
        op = Operator.sorted(h, args.p)
        r = block_krylov(op, k, block=b, seed=step)
        e1.record()
        torch.cuda.synchronize()
        if step >= args.warmup:
            times.append(e0.elapsed_time(e1))
            infos.append(r.info)
        AZ = fp64_product(op, r.Z)
        res = (torch.linalg.vector_norm(AZ - r.Z * r.lam[None, :], dim=0) / r.sigma).cpu().tolist()
        l1.l1dm_free(h)
    ms = statistics.mean(times)
    upd = n * d * r.columns
    pm = statistics.mean(i["product_ms"] for i in infos)
    tm = statistics.mean(i["total_ms"] for i in infos)
    print(json.dumps({
        "metric": "block-Krylov top-k singular values of the l1 distance matrix (NEXT-2)",
        "value": upd / (ms * 1e-3), "unit": "updates/s (n*d*columns through the products)",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "dtype": "f64 accumulation over f32 inputs (hi|lo split)",
        "data": "synthetic", "config": {"workload": args.workload, "n": n, "d": d, "k": k,
                                        "block": b, "depth": r.info["depth"],
                                        "products": r.products, "columns": r.columns,
                                        "p": args.p},
        "krylov_ms": tm, "products_ms": pm, "products_share_of_krylov": pm / tm,
        "dense_ms": tm - pm, "prepare_plus_krylov_ms": ms,
        "sigma_top": r.sigma[:min(k, 8)].cpu().tolist(), "ritz_residuals": res[:min(k, 8)],
    }))
    return 0


def main_l2approx(args):
    """NEXT-3 measurement (1 GPU): a step = embed (Thm. l2embed GEMM) + l1 prepare on the k
    embedded coordinates + the workload's queries.  value = n k m queries / step time."""
    import paper_2210_15114_b200 as l1
    from paper_2210_15114_b200 import workloads as wl
    from paper_2210_15114_b200.l2approx import L2Approx
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = wl.workload(args.workload)
    Q = args.queries or w.queries
    X = wl.make_points(w, dev)
    Zs = [wl.make_query(w, t, dev) for t in range(Q if w.fresh_queries else 1)]
    Y = torch.empty((w.n, w.m), dtype=torch.float64, device=dev)
    times, embed_ms = [], []
    k = None
    for step in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        eng = L2Approx(X, eps=args.l2approx, seed=step)
        e1.record()
        for q in range(Q):
            eng.matvec(Zs[q % len(Zs)], Y)
        e2.record()
        torch.cuda.synchronize()
        k = eng.k
        eng.close()
        if step >= args.warmup:
            times.append(e0.elapsed_time(e2))
            embed_ms.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    print(json.dumps({
        "metric": "approximate l2 distance-matrix product via the l1 engine (NEXT-3)",
        "value": w.n * k * w.m * Q / (ms * 1e-3), "unit": "updates/s (n*k*m on the embedding)",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "dtype": "f64 accumulation over f32 inputs", "data": "synthetic",
        "config": {"workload": args.workload, "n": w.n, "d": w.d, "m": w.m, "eps": args.l2approx,
                   "k": k, "queries_per_step": Q},
        "embed_plus_prepare_ms": statistics.mean(embed_ms),
        "query_ms": (ms - statistics.mean(embed_ms)) / Q}))
    return 0


if __name__ == "__main__":
    a = parse()
    if a.l2approx > 0 and a.impl == "ours":
        sys.exit(main_l2approx(a))
    if a.krylov > 0 and a.impl == "ours":
        sys.exit(main_krylov(a))
    sys.exit(run_reference(a) if a.impl == "reference" else main_ours(a))
