#!/bin/bash
# Profiling recipe (run under gpurun on one B200; outputs land in gpurun_out/).
#   1. the bench command itself, plain (must exit 0 before any ncu run)
#   2. ncu launch list of the same command (gpu__time_duration per launch, clocks not locked)
#   3. ncu --set full of the query's top kernels (one launch each) for DRAM traffic
# usage: profiles/run_profile.sh <workload> [kernel-regex]
set -e
W=${1:-c3}
K=${2:-"k5_scan|k6_accumulate"}
CMD="python bench.py --workload $W --steps 1 --warmup 1 --queries 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$W.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/prof_launches_$W.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$K" \
    -s 4 -c 3 -o gpurun_out/full_$W $CMD > gpurun_out/prof_full_$W.log 2>&1
