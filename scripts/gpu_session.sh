set -x
timeout 900 python scripts/soft_timing.py C2,C3,C4 > gpurun_out/softtime.log 2>&1
