timeout 3000 env CG_LIB=$PWD/paper_2601_17026_b200/libcolgraph_dbg.so python -m pytest tests -m gpu -q -x -k "not limits" > gpurun_out/s14_dbg_tests.log 2>&1
tail -3 gpurun_out/s14_dbg_tests.log
