set -x
timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_soft.py tests/test_gpu_slabs.py -x -q > gpurun_out/t_flow.log 2>&1
