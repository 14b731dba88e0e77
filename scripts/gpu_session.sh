set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1 || exit 2
timeout 400 python bench.py > gpurun_out/bench.log 2>&1 || exit 3
timeout 120 python scripts/profile_one.py C4 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_one.py C4 > gpurun_out/ncu_list.log 2>&1 || exit 4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 4 -c 3 -o gpurun_out/prof_walk python scripts/profile_one.py C4 > gpurun_out/ncu_full.log 2>&1 || exit 5
