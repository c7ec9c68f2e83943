for w in c4 c5; do
  timeout 300 python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --queries 3 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w', 'k5', d['query_ms'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
  L1DM_GATHER_SEQ=1 timeout 300 python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --queries 3 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$w', 'seq', d['query_ms'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
L1DM_GATHER_SEQ=1 timeout 300 python bench.py --workload c3 --mode gather --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --queries 3 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3g', 'seq', d['query_ms'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
L1DM_GATHER_SEQ=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size" 2>&1 | tail -2
