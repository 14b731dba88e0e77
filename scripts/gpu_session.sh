set -x
timeout 120 ./bench_tools/random_gather > gpurun_out/random_gather.json 2>&1
