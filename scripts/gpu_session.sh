set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/t_smoke.log 2>&1 || exit 1
CG_TRACE=1 timeout 60 python scripts/diag_solve.py C4 > gpurun_out/t_diag4.log 2> gpurun_out/t_trace4.log || exit 5
timeout 1200 python scripts/ab.py C3,C4,C5 3 'bitmap:' > gpurun_out/t_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/t_tests.log 2>&1 || exit 3
