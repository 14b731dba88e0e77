set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/t_smoke.log 2>&1 || exit 1
timeout 900 python scripts/ab.py C3,C4,C5 3 'base:' 'relist:CG_RELIST=1' > gpurun_out/t_ab.log 2>&1
CG_RELIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or c1 or c2 or full_size" > gpurun_out/t_tests.log 2>&1 || exit 3
