true
for v in kg48 kg96 u12 u24 u32 kg32u16; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rs_$v.log 2>&1; done
