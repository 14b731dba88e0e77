set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/t_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_flow.py -x -q > gpurun_out/t_flow.log 2>&1 || exit 2
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_size" > gpurun_out/t_tests.log 2>&1 || exit 3
