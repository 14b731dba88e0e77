set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1 || exit 3
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python scripts/diag_solve.py > gpurun_out/diag.log 2>&1
timeout 300 python scripts/flow_export_timing.py C3,C4,C5 > gpurun_out/flowtime.log 2>&1
timeout 600 python scripts/soft_timing.py C2,C3,C4 > gpurun_out/softtime.log 2>&1
timeout 120 python scripts/profile_one.py C4 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_one.py C4 > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 4 -c 3 -o gpurun_out/prof_walk python scripts/profile_one.py C4 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bfs_run -s 3 -c 1 -o gpurun_out/prof_bfs python scripts/profile_one.py C4 > gpurun_out/ncu_full2.log 2>&1
