timeout 300 python scratch/scat.py c3 auto
L1DM_REDUCE_ALL_ASYNC=0 timeout 300 python scratch/scat.py c3 auto
timeout 300 python scratch/scat.py c3 auto
