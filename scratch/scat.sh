for r in 0 1 2; do for a in 0 1 2; do echo "R=$r A=$a"; L1DM_ZPOL_R=$r L1DM_ZPOL_A=$a timeout 300 python scratch/scat.py c3 auto; done; done
