unset L1DM_LIB; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ra_t2.log 2>&1
for v in t4 t8; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ra_$v.log 2>&1; done
