set -x
CG_LIB=paper_2601_17026_b200/libcolgraph_dbg.so timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_dbg_tests.log 2>&1
echo rc=$? >> gpurun_out/t_dbg_tests.log
