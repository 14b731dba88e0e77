set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/t_smoke.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_aniso.py tests/test_gpu_flow.py -x -q > gpurun_out/t_aniso.log 2>&1 || exit 2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1 || exit 3
timeout 300 python scripts/flow_export_timing.py C3,C4 > gpurun_out/t_flowtime.log 2>&1 || exit 4
