"""bench.py's JSON-line contract on the small c1 workload: the reference arm (the CPU oracle,
runs anywhere), our arm at N = 1, and a dry run of the N = 2 path as two processes sharing one
GPU with gloo collectives (the NCCL-collective path's kernels never wait on each other)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run(args, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
             "--warmup", "1"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "updates/s"
    assert d["higher_is_better"] is True and d["config"]["workload"] == "c1"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def check_ours(d, n_gpus):
    assert d["n_gpus"] == n_gpus and d["value"] > 0 and d["ms_per_step"] > 0
    for k in ("metric", "unit", "steps", "warmup", "higher_is_better", "scaling", "dtype", "data",
              "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac"} <= set(r)
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # the timed work is validated (queries 0 and Q-1) and the inputs hashed
    assert d["parity"]["pass"] and d["parity"]["max_col_rel_l2"] <= 1e-9
    assert len(d["parity"]["queries"]) == 2 and d["parity"]["rows"] >= 4
    assert len(d["inputs_sha256"]["X"]) == 64


@pytest.mark.gpu
def test_ours_single_gpu_line():
    d = run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3",
             "--no-cpu-baseline"])
    check_ours(d, 1)


@pytest.mark.gpu
def test_ours_two_rank_dry_run_line():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
             "--workload", "c1", "--steps", "3", "--warmup", "3"],
            env={"L1DM_BENCH_DEVICE": "0", "L1DM_BENCH_BACKEND": "gloo"})
    check_ours(d, 2)
    assert d["config"]["parallelism"] == "coord-shard x2"
    mg = d["multi_gpu"]
    assert mg["compute_only_ms_per_query"] > 0 and mg["collective_alone_ms"] > 0
    assert mg["message_bytes"] == 2048 * 1 * 8
