for p in 2 4 6; do
  unset L1DM_LIB; timeout 600 python bench.py --p $p --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/e2_p$p.log 2>&1
  L1DM_LIB=$PWD/scratch/libl1dm_e4.so timeout 600 python bench.py --p $p --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/e4_p$p.log 2>&1
done
