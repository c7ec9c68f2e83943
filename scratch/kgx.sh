for v in def kgx64 kgx96 def2; do
  if [ ${v#def} != $v ]; then unset L1DM_LIB; else export L1DM_LIB=$PWD/scratch/libl1dm_$v.so; fi
  timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/kgx_$v.log 2>&1
  timeout 600 python bench.py --workload c5 --p 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/kgx_p3_$v.log 2>&1
done
