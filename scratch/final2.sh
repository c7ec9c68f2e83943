B="timeout 900 python bench.py"
$B > gpurun_out/f_c3.log 2>&1
$B --impl reference > gpurun_out/f_c3_reference.log 2>&1
$B --workload c2 --steps 10 > gpurun_out/f_c2.log 2>&1
$B --workload c4 --steps 2 > gpurun_out/f_c4.log 2>&1
$B --workload c5 --steps 3 > gpurun_out/f_c5.log 2>&1
$B --p 3 --steps 2 --no-cpu-baseline > gpurun_out/f_c3_p3.log 2>&1
$B --p 2 --steps 3 --no-cpu-baseline > gpurun_out/f_c3_p2.log 2>&1
$B --workload c5 --p 3 --steps 2 --no-cpu-baseline > gpurun_out/f_c5_p3.log 2>&1
$B --krylov 16 --steps 2 --no-cpu-baseline > gpurun_out/f_c3_krylov16.log 2>&1
$B --l2approx 0.5 --steps 2 --no-cpu-baseline > gpurun_out/f_c3_l2approx05.log 2>&1
bash profiles/run_profile.sh c3 "k5_scan_seq|k5_reduce_all"
