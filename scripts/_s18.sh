timeout 1500 python scripts/ab.py C5,C3 5 'base:' 'tail8:CG_TAIL_BATCH=8' 'base2:' 'tail8b:CG_TAIL_BATCH=8' > gpurun_out/s18_ab.txt 2>&1
