for v in "1 16384" "1 4096" "1 65536" "0 0"; do
  set -- $v
  export L1DM_RUNS_AGG=$1 L1DM_RUNS_AGG_CHUNK=$2
  timeout 600 python -m pytest tests/test_gpu_runs.py -q -x > gpurun_out/pytest_ra_$1_$2.log 2>&1
  timeout 600 python bench.py --workload c5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ra_c5_$1_$2.log 2>&1
done
