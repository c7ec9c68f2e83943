unset L1DM_LIB; timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ev_default.log 2>&1
for v in e2 e8 e16; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ev_$v.log 2>&1; done
