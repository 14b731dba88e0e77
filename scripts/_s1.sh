set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 300 env CG_TRACE=1 python scripts/diag_solve.py C4 > gpurun_out/s1_trace_c4.txt 2>&1
timeout 1500 python scripts/relabel_study.py C4 100,400,800 > gpurun_out/s1_study_c4.jsonl 2> gpurun_out/s1_study_c4.err
timeout 1200 python scripts/relabel_study.py C5 2000,9000 > gpurun_out/s1_study_c5.jsonl 2> gpurun_out/s1_study_c5.err
