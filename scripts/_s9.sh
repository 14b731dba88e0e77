timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s9_gpu_all.log 2>&1
timeout 600 env CG_TRACE=1 python scripts/slab_overhead.py C4 > gpurun_out/s9_slabs_default.jsonl 2> gpurun_out/s9_slabs_default.err
timeout 400 python bench.py > gpurun_out/s9_bench.log 2>&1
tail -3 gpurun_out/s9_gpu_all.log
