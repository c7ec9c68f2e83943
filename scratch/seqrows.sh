unset L1DM_LIB; timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sr_default.log 2>&1
for v in r512 r2048; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sr_$v.log 2>&1; done
for v in r512 r2048; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python -m pytest tests/test_gpu_scatter.py -q -x > gpurun_out/pytest_sr_$v.log 2>&1; done
