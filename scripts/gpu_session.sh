set -x
timeout 600 python -m pytest tests/test_gpu_limits.py -x -q -s > gpurun_out/t_limits.log 2>&1
echo rc=$? >> gpurun_out/t_limits.log
