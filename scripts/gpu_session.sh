set -x
timeout 900 python -m pytest tests/test_gpu_soft.py -x -q > gpurun_out/t_soft.log 2>&1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py -x -q -k "not full_size" > gpurun_out/t_slabs.log 2>&1
timeout 600 python scripts/ab.py C4 3 'hard:' > gpurun_out/t_ab.log 2>&1
