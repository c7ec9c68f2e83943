timeout 300 python scratch/scat.py c3 auto
timeout 300 python scratch/scat.py c3 auto
