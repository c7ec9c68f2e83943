export PYTHONPATH=$PWD
timeout 300 python scratch/sortbench.py hint > gpurun_out/sortbench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k3_rank -c 2 --csv --log-file gpurun_out/k3.csv python scratch/prep1.py c4 > /dev/null 2>&1
