for v in 1 0; do
  export L1DM_RUNS_GATHER=$v
  timeout 600 python -m pytest tests/test_gpu_runs.py -q -x > gpurun_out/pytest_runs_$v.log 2>&1
  timeout 600 python bench.py --workload c5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rg_c5_$v.log 2>&1
done
