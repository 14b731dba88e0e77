set -x
timeout 1800 python scripts/ab.py C3,C4,C5 3 'default:' 'workonly:CG_GR_BETA=1000' 'ws_workonly:CG_GR_BETA=1000,CG_WALK_WS=1' 'ws_b2:CG_GR_BETA=2,CG_WALK_WS=1' > gpurun_out/t_ab.log 2>&1
