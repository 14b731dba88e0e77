set -x
timeout 900 python -m pytest tests/test_gpu_soft.py -x -q > gpurun_out/t_soft.log 2>&1
timeout 600 python scripts/soft_timing.py C2,C3,C4 > gpurun_out/softtime.log 2>&1
timeout 600 python scripts/ab.py C4 3 'hard:' > gpurun_out/t_ab.log 2>&1
