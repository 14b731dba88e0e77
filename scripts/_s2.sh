set -x
python -m paper_2601_17026_b200.build
timeout 900 python -m pytest tests/test_gpu_relabel.py -x -q > gpurun_out/s2_relabel.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nccl_loopback.py -x -q > gpurun_out/s2_loopback.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gap.py -x -q > gpurun_out/s2_gap.log 2>&1
timeout 300 env CG_TRACE=1 python scripts/diag_solve.py C4 > gpurun_out/s2_trace_c4.txt 2>&1
timeout 300 python scripts/diag_solve.py C3,C4,C5 > gpurun_out/s2_diag.jsonl 2>&1
timeout 300 env CG_RELABEL=bfs python scripts/diag_solve.py C3,C4,C5 > gpurun_out/s2_diag_bfs.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_gpu_all.log 2>&1
tail -3 gpurun_out/s2_*.log
