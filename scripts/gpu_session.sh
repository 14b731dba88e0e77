set -x
timeout 1500 python scripts/ab.py C4 6 'default:' 'ws:CG_WALK_WS=1' 'g2ws:CG_LIB=paper_2601_17026_b200/libcolgraph_gather2.so,CG_WALK_WS=1' > gpurun_out/t_ab.log 2>&1
timeout 900 python scripts/ab.py C3,C5 3 'default:' 'ws:CG_WALK_WS=1' 'g2ws:CG_LIB=paper_2601_17026_b200/libcolgraph_gather2.so,CG_WALK_WS=1' >> gpurun_out/t_ab.log 2>&1
