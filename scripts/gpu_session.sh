set -x
timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_aniso.py -x -q > gpurun_out/t_flow.log 2>&1 || exit 2
timeout 300 python scripts/flow_export_timing.py C2,C3,C4,C5 > gpurun_out/t_flowtime.log 2>&1 || exit 4
