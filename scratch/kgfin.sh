timeout 900 python -m pytest tests/test_gpu_runs.py tests/test_gpu_lp.py tests/test_gpu_peer.py -x -q > gpurun_out/kgfin_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --workload c5 > gpurun_out/kgfin_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --workload c5 --p 3 --no-cpu-baseline > gpurun_out/kgfin_c5p3.log 2>&1; echo c5p3=$?
