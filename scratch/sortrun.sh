export PYTHONPATH=$PWD
timeout 300 python scratch/sortbench.py rts >> gpurun_out/sortbench.log 2>&1
L1DM_SORT_ONESWEEP=1 timeout 300 python scratch/sortbench.py onesweep >> gpurun_out/sortbench.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
