unset L1DM_LIB; timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m1_default.log 2>&1
for v in i8m4 i8m5 i8m6 i8m7 i4m6; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m1_$v.log 2>&1; done
