# ad-hoc GPU session (gpurun): stops at the first failing step
set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/t_smoke.log 2>&1 || exit 1
CG_TILE_PROF=1 CG_TRACE=1 timeout 100 python scripts/diag_solve.py C4 > gpurun_out/t_diag_a.log 2> gpurun_out/t_trace4.log || exit 5
CG_TILE_PROF=1 CG_TRACE=1 CG_TILE_RELABEL=-1 timeout 100 python scripts/diag_solve.py C4 > gpurun_out/t_diag_b.log 2> gpurun_out/t_trace4_r0.log || exit 5
CG_TILE_PROF=1 CG_TRACE=1 CG_TILE_STEPS=16 timeout 100 python scripts/diag_solve.py C4 > gpurun_out/t_diag_c.log 2> gpurun_out/t_trace4_s16.log || exit 5
CG_SWEEP=2 CG_TRACE=1 timeout 100 python scripts/diag_solve.py C4 > gpurun_out/t_diag_d.log 2> gpurun_out/t_trace4_old.log || exit 5
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "worked or tiny or c1 or c2 or edge or constant" > gpurun_out/t_tests.log 2>&1 || exit 3
