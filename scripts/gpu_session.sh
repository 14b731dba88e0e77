set -x
timeout 900 python scripts/ab.py C3,C4,C5 3 'aos:' 'soa:CG_LIB=paper_2601_17026_b200/libcolgraph_soa.so' > gpurun_out/t_ab.log 2>&1
