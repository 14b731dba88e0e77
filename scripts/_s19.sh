timeout 900 python -m pytest tests/test_gpu_relabel.py tests/test_gpu_variants.py -x -q -k "bottomup or BU or labels" > gpurun_out/s19_tests.log 2>&1
timeout 1500 python scripts/ab.py C3,C4,C5 2 'base:' 'bu4_1m:CG_BFS_BU=4,1000000' 'bu2_1m:CG_BFS_BU=2,1000000' 'bu8_500k:CG_BFS_BU=8,500000' 'bu16_250k:CG_BFS_BU=16,250000' > gpurun_out/s19_ab.txt 2>&1
timeout 200 env CG_TRACE=1 CG_BFS_BU=4,1000000 python scripts/diag_solve.py C4 > gpurun_out/s19_trace_c4.txt 2>&1
tail -2 gpurun_out/s19_tests.log
