timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1
B="timeout 900 python bench.py"
$B > gpurun_out/r_c3.log 2>&1
$B --impl reference > gpurun_out/r_c3_ref.log 2>&1
$B --workload c2 --steps 10 > gpurun_out/r_c2.log 2>&1
$B --workload c5 --steps 3 > gpurun_out/r_c5.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
