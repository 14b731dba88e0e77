set -x
CG_LIB=paper_2601_17026_b200/libcolgraph_dbg.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_dbg_tests.log 2>&1
echo rc=$? >> gpurun_out/t_dbg_tests.log
