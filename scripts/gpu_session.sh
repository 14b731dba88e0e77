# One GPU session's evidence (run under gpurun from the repo root; then
# `python scripts/save_profiles.py <tag>` here copies it into profiles/).
set -x
timeout 60 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1 || exit 3
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python scripts/diag_solve.py > gpurun_out/diag.log 2>&1
# relabel schedule of an unprofiled C4 solve, replayed under ncu (CG_GR_SCHEDULE) so the
# profiled runs take the same trajectory as the bench instead of the replay-slowed one
rm -f gpurun_out/grlog.txt
CG_GR_LOG=gpurun_out/grlog.txt timeout 120 python scripts/profile_one.py C4 > gpurun_out/plain.log 2>&1
export CG_GR_SCHEDULE=$(head -1 gpurun_out/grlog.txt)
# launch list of the bench command itself (cold-cache, serialised: shares, not absolutes)
timeout 900 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
# DRAM bytes of every sweep launch of one C4 solve + that solve's algorithmic bytes
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"k_walk_ws|k_sweep_v" --csv --log-file gpurun_out/sweep_traffic.csv \
  python scripts/profile_one.py C4 > gpurun_out/sweep_traffic.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_walk_ws -s 4 -c 3 -o gpurun_out/prof_walk python scripts/profile_one.py C4 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bfs_run -s 3 -c 1 -o gpurun_out/prof_bfs python scripts/profile_one.py C4 > gpurun_out/ncu_full2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bfs2_init|k_colgr_rebuild" -s 2 -c 2 -o gpurun_out/prof_passes python scripts/profile_one.py C4 > gpurun_out/ncu_full3.log 2>&1
tail -1 gpurun_out/gpu_tests.log; cat gpurun_out/bench.log | tail -1
