L1DM_SCATTER_MB=8 timeout 300 python scratch/scat.py c3 scatter
L1DM_SCATTER_MB=4 timeout 300 python scratch/scat.py c3 scatter
L1DM_SCATTER_MB=16 timeout 300 python scratch/scat.py c3 scatter
