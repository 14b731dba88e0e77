set -x
timeout 600 python -m pytest tests/test_gpu_soft.py -x -q -k full_size > gpurun_out/t_soft_full.log 2>&1
timeout 600 python scripts/soft_timing.py C2,C3,C4 > gpurun_out/t_soft_time.log 2>&1
