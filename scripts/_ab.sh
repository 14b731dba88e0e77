P=$PWD/paper_2601_17026_b200
CG_LIB=$P/libcolgraph_bfs_r1m2.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not full" 2>&1 | tail -1
CG_LIB=$P/libcolgraph_bfs_r4m1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not full" 2>&1 | tail -1
timeout 1800 python scripts/ab.py C3,C4,C5 3 'def:' "r1m2:CG_LIB=$P/libcolgraph_bfs_r1m2.so" "r2m2:CG_LIB=$P/libcolgraph_bfs_r2m2.so" "r4m1:CG_LIB=$P/libcolgraph_bfs_r4m1.so"
