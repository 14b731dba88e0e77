timeout 600 python scripts/diag_solve.py > gpurun_out/diag.log 2>&1
