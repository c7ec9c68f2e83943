"""Summarise ncu outputs into profiles/: per-kernel launch shares and full-capture metrics.

    python profiles/summarize.py <workload> <launches.csv> <full.ncu-rep> <round-tag>
"""
import collections
import csv
import json
import subprocess
import sys

w, launches, rep, tag = sys.argv[1:5]
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1}.get(r[ui], 1)
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale
# shares over the library's kernels (l1dm::); torch's kernels (the inputs' RNG and the bench's
# after-the-timed-region parity check, definition in fp64) are listed apart
lib = {k: v for k, v in agg.items() if k.startswith("l1dm::")}
tot = sum(v[1] for v in lib.values())
out = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
       f"# workload {w}: bench.py --workload {w} --steps 1 --warmup 1 --queries 3 (profiles/run_profile.sh)",
       f"# share = of the library's (l1dm::) kernel time {tot:.3f} ms",
       f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
for k, v in sorted(lib.items(), key=lambda x: -x[1][1]):
    out.append(f"{k[:60]:60s} {v[0]:8d} {v[1]:10.3f} {v[1] / tot * 100:6.1f}%")
other = {k: v for k, v in agg.items() if not k.startswith("l1dm::")}
if other:
    out.append("# not the library's (input generation, parity check after the timed region):")
    for k, v in sorted(other.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:60]:60s} {v[0]:8d} {v[1]:10.3f}")
open(f"profiles/{tag}_{w}_launch_shares.txt", "w").write("\n".join(out) + "\n")
if rep == "-":  # launch list only
    sys.exit(0)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__t_sectors.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
lines = [f"# ncu --set full --clock-control none, workload {w}, one launch per kernel", ""]
traffic = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    lines.append("== " + name[:100])
    for k in keys:
        if k in hdr:
            lines.append(f"   {k:60s} {r[hdr.index(k)]:>18s} {units[hdr.index(k)]}")
    for i, h in enumerate(hdr):
        if "warps_issue_stalled" in h and "per_issue_active.ratio" in h:
            try:
                if float(r[i]) > 0.5:
                    lines.append(f"   stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):54s} {r[i]:>18s}")
            except ValueError:
                pass
    sc = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rb = float(r[hdr.index("dram__bytes_read.sum")]) * sc[units[hdr.index("dram__bytes_read.sum")]]
    wb = float(r[hdr.index("dram__bytes_write.sum")]) * sc[units[hdr.index("dram__bytes_write.sum")]]
    if "k5_scan_lb" in name:  # scatter mode, single pass: the apply (timing kind accumulate)
        kind = "scatter_accumulate"
    elif "k5_reduce_all" in name:  # scatter mode: tile totals of every column (timing kind scan)
        kind = "scatter_scan"
    elif "k5_scan_seq" in name:  # scatter mode: <mb, 0> reduce (timing kind scan), <mb, 1> apply
        kind = "scatter_accumulate" if ", 1>" in name or ",1>" in name else "scatter_scan"
    elif "k20_runs_hist" in name:  # runs mode: the histogram (timing kind scan)
        kind = "runs_scan"
    elif "k22_runs" in name:  # runs mode: the expansion (timing kind accumulate)
        kind = "runs_accumulate"
    elif "k5_scan" in name or "k6_accumulate" in name:
        kind = "gather_" + ("scan" if "scan" in name else "accumulate")
    else:
        kind = name.split("(")[0]
    traffic.setdefault(kind, rb + wb)
open(f"profiles/{tag}_{w}_ncu_full.txt", "w").write("\n".join(lines) + "\n")
out_json = f"profiles/ncu_traffic_{w}.json"
try:
    old = json.load(open(out_json))
except Exception:
    old = {}
old.pop("scan", None)
old.pop("accumulate", None)
sources = old.pop("sources", {})
for k in traffic:
    sources[k] = f"profiles/{tag}_{w}_ncu_full.txt"
json.dump({**{k: v for k, v in old.items() if k not in ("unit", "source")}, **traffic,
           "unit": "bytes per launch (dram read+write)", "sources": sources},
          open(out_json, "w"), indent=1)
print("\n".join(out))
print(json.dumps(traffic, indent=1))
