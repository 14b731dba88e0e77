set -x
timeout 1500 python scripts/ab.py C3,C4,C5 3 'minb4:' 'minb6:CG_LIB=paper_2601_17026_b200/libcolgraph_minb6.so' 'minb8:CG_LIB=paper_2601_17026_b200/libcolgraph_minb8.so' > gpurun_out/t_ab.log 2>&1
