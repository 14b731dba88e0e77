CG_BFS_TRUNC=16384,16 CG_TRACE=1 timeout 120 python scripts/profile_one.py C3 > gpurun_out/trace_C3_t16k.txt 2>&1
CG_BFS_TRUNC=16384,16 CG_TRACE=1 timeout 120 python scripts/profile_one.py C4 > gpurun_out/trace_C4_t16k.txt 2>&1
timeout 1500 python scripts/ab.py C3,C4,C5 4 'base:' 't16k_4:CG_BFS_TRUNC=16384;4' 't16k_8:CG_BFS_TRUNC=16384;8' 't64k_16:CG_BFS_TRUNC=65536;16' 't64k_4:CG_BFS_TRUNC=65536;4' 't128k_8:CG_BFS_TRUNC=131072;8' 't4k_8:CG_BFS_TRUNC=4096;8' 't16k_32:CG_BFS_TRUNC=16384;32' 'base2:' > gpurun_out/ab_trunc2.txt 2>&1
cat gpurun_out/ab_trunc2.txt
