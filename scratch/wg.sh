timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/wg_c4.log 2>&1
timeout 600 python bench.py --workload c3 --mode gather --steps 1 --warmup 1 --queries 5 --no-cpu-baseline --no-e2e > gpurun_out/wg_c3g.log 2>&1
