set -x
timeout 900 python -m pytest tests/test_gpu_relabel.py -x -q > gpurun_out/s4_tests.log 2>&1
timeout 300 env CG_TRACE=1 python scripts/diag_solve.py C4 > gpurun_out/s4_trace_c4.txt 2>&1
timeout 300 python scripts/diag_solve.py C2,C3,C4,C5 > gpurun_out/s4_diag.jsonl 2>&1
tail -n 3 gpurun_out/s4_tests.log
