unset L1DM_LIB; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/su_default.log 2>&1
for v in u8 u2 u16; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/su_$v.log 2>&1; done
for v in u8 u16; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --p 3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/su3_$v.log 2>&1; done
timeout 600 python bench.py --p 3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/su3_default.log 2>&1
