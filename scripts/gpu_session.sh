timeout 1200 python scripts/slab_overhead.py C3,C4 > gpurun_out/slab_overhead.jsonl 2>&1
