timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
for v in 1 0; do
  export L1DM_BULK_GATHER=$v
  timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/bk_c4_$v.log 2>&1
  timeout 600 python bench.py --workload c3 --mode gather --steps 1 --warmup 1 --queries 5 --no-cpu-baseline --no-e2e > gpurun_out/bk_c3g_$v.log 2>&1
  timeout 600 python bench.py --workload c5 --mode gather --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/bk_c5g_$v.log 2>&1
done
