CG_BFS_TRUNC=16384,8 CG_TRACE=1 timeout 120 python scripts/profile_one.py C3 > gpurun_out/trace_C3_t16k_q.txt 2>&1
timeout 1500 python scripts/ab.py C2,C3,C4,C5 4 'base:' 't16k_8:CG_BFS_TRUNC=16384;8' 't16k_4:CG_BFS_TRUNC=16384;4' 't64k_16:CG_BFS_TRUNC=65536;16' 't64k_8:CG_BFS_TRUNC=65536;8' 't32k_8:CG_BFS_TRUNC=32768;8'  't16k_8_old:CG_BFS_TRUNC=16384;8;0' 'base2:' > gpurun_out/ab_trunc3.txt 2>&1
cat gpurun_out/ab_trunc3.txt
