set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/re_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/re_bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/re_ref.log 2>&1; echo ref=$?
