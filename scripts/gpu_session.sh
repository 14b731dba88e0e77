set -x
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
