set -x
timeout 900 python -m pytest tests/test_gpu_soft.py tests/test_gpu_flow.py -x -q > gpurun_out/t_soft.log 2>&1
