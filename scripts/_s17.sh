timeout 1500 python scripts/ab.py C5,C3,C4 2 'base:' 'tail4:CG_TAIL_BATCH=4' 'tail8:CG_TAIL_BATCH=8' 'tail16:CG_TAIL_BATCH=16' 'tail32:CG_TAIL_BATCH=32' > gpurun_out/s17_ab.txt 2>&1
