timeout 1500 python scripts/ab.py C5,C4 2 'base:' 'wm0:CG_WALK_MIN=0' 'wm0k256:CG_WALK_MIN=0,CG_WALK=256' 'wm0k1024:CG_WALK_MIN=0,CG_WALK=1024' 'wm1e4:CG_WALK_MIN=1e-4' 'wm1e5k256:CG_WALK_MIN=1e-5,CG_WALK=256' > gpurun_out/s16_ab.txt 2>&1
timeout 300 env CG_TRACE=1 CG_WALK_MIN=0 python scripts/diag_solve.py C5 > gpurun_out/s16_trace_c5_wm0.txt 2>&1
timeout 300 env CG_TRACE=1 python scripts/diag_solve.py C5 > gpurun_out/s16_trace_c5.txt 2>&1
