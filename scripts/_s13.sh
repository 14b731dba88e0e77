timeout 900 python -m pytest tests/test_gpu_relabel.py tests/test_gpu_variants.py -x -q -k "trunc or labels" > gpurun_out/s13_tests.log 2>&1
timeout 1200 python scripts/ab.py C3,C4,C5 2 'base:' 't64_16:CG_BFS_TRUNC=64,16' 't256_32:CG_BFS_TRUNC=256,32' 't2k_64:CG_BFS_TRUNC=2048,64' 't16k_128:CG_BFS_TRUNC=16384,128' 't2k_16:CG_BFS_TRUNC=2048,16' > gpurun_out/s13_ab.txt 2>&1
timeout 200 env CG_TRACE=1 CG_BFS_TRUNC=2048,64 python scripts/diag_solve.py C4 > gpurun_out/s13_trace_c4.txt 2>&1
tail -2 gpurun_out/s13_tests.log
