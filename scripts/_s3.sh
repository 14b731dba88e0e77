timeout 1500 python scripts/ab.py C3,C4,C5 4 'base:' 't64_16:CG_BFS_TRUNC=64;16' 't256_32:CG_BFS_TRUNC=256;32' 't2k_64:CG_BFS_TRUNC=2048;64' 't2k_16:CG_BFS_TRUNC=2048;16' 't16k_64:CG_BFS_TRUNC=16384;64' 't16k_16:CG_BFS_TRUNC=16384;16' 'base2:' > gpurun_out/ab_trunc.txt 2>&1
cat gpurun_out/ab_trunc.txt
