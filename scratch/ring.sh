timeout 600 python -m pytest tests/test_gpu_sortfree.py tests/test_gpu_l2approx.py -q -x > gpurun_out/pytest_sf.log 2>&1
for v in 1 0; do
  export L1DM_K12_RING=$v
  for p in 2 4; do timeout 600 python bench.py --p $p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ring_${v}_p$p.log 2>&1; done
done
