timeout 1200 python -m pytest tests/test_gpu_next3.py -x -q > gpurun_out/s10_next3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_flow.py tests/test_gpu_aniso.py tests/test_gpu_soft.py tests/test_gpu_relabel.py tests/test_gpu_variants.py -x -q > gpurun_out/s10_others.log 2>&1
timeout 300 python scripts/diag_solve.py C3,C4,C5 > gpurun_out/s10_diag.jsonl 2>&1
tail -3 gpurun_out/s10_next3.log gpurun_out/s10_others.log
