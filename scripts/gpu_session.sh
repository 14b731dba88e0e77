set -x
timeout 300 python scripts/phase_timing.py C4 16 > gpurun_out/t_phase.log 2>&1
