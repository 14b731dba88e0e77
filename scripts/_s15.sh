timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s15_gpu_all.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s15_bench.log 2>&1
timeout 300 python scripts/diag_solve.py > gpurun_out/s15_diag.jsonl 2>&1
tail -3 gpurun_out/s15_gpu_all.log
