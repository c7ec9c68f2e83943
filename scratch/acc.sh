unset L1DM_LIB; timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/acc_default.log 2>&1
for v in a4 a16; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --queries 3 --no-cpu-baseline --no-e2e > gpurun_out/acc_$v.log 2>&1; done
