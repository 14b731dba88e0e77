L=paper_2601_17026_b200
timeout 1200 python scripts/ab.py C3,C4,C5 2 'base:' 'small0:CG_BFS_SMALL=0' 'small16:CG_BFS_SMALL=16' 'small256:CG_BFS_SMALL=256' 'bar256:CG_BAR_NS=256' 'bar128:CG_BAR_NS=128' "nopre:CG_LIB=$PWD/$L/libcolgraph_nopre.so" "bfs2:CG_LIB=$PWD/$L/libcolgraph_bfs2.so" > gpurun_out/s12_ab.txt 2>&1
timeout 200 env CG_TRACE=1 python scripts/diag_solve.py C4 > gpurun_out/s12_trace_c4.txt 2>&1
