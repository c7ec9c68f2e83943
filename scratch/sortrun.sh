export PYTHONPATH=$PWD
timeout 300 python scratch/sortbench.py default >> gpurun_out/sortbench.log 2>&1
for v in i8m3 i8m4 i12m3 i16m2; do L1DM_LIB=$PWD/scratch/libl1dm_$v.so timeout 300 python scratch/sortbench.py $v >> gpurun_out/sortbench.log 2>&1; done
