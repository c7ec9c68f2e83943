unset L1DM_LIB; timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/fp_0.log 2>&1
L1DM_LIB=$PWD/scratch/libl1dm_fp.so timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/fp_1.log 2>&1
L1DM_LIB=$PWD/scratch/libl1dm_fp.so timeout 600 python -m pytest tests/test_gpu_sortfree.py -q -x > gpurun_out/pytest_fp.log 2>&1
