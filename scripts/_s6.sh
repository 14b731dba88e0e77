timeout 200 env CG_TRACE=1 python scripts/diag_solve.py C4 > gpurun_out/s6_trace_c4.txt 2>&1
timeout 900 python scripts/ab.py C3,C4,C5 3 'base:' 'full:CG_BFS_FULL=1' 'recbfs:CG_RELABEL=bfs' 'gap1:AB_OPTS={"gap_every":1}' 'gap4:AB_OPTS={"gap_every":4}' 'walk256:CG_WALK=256' 'ce8:AB_OPTS={"check_every":8}' 'beta05:CG_GR_BETA=0.5' 'beta2:CG_GR_BETA=2' > gpurun_out/s6_ab.txt 2>&1
