set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
for v in default s64 s48; do
  if [ $v = default ]; then unset L1DM_LIB; else export L1DM_LIB=$PWD/scratch/libl1dm_$v.so; fi
  timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/c4_$v.log 2>&1
  timeout 600 python bench.py --workload c3 --mode gather --steps 1 --warmup 1 --queries 5 --no-cpu-baseline --no-e2e > gpurun_out/c3g_$v.log 2>&1
  timeout 600 python bench.py --workload c5 --mode gather --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/c5g_$v.log 2>&1
done
