unset L1DM_LIB; timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/k14_default.log 2>&1
for v in g2k32 g4k16 g4k32; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --p 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/k14_$v.log 2>&1; done
