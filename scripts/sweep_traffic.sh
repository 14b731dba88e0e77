# Per-launch DRAM bytes of EVERY sweep launch (k_walk / k_sweep_v) of one C4 solve, next to
# the same solve's algorithmic bytes (profile_one.py prints sweep_bytes_alg).
set -e
timeout 300 python scripts/profile_one.py C4 > gpurun_out/profile_one_plain.log 2>&1
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"k_walk|k_sweep_v" --csv --log-file gpurun_out/sweep_traffic.csv \
  python scripts/profile_one.py C4 > gpurun_out/sweep_traffic.log 2>&1
tail -2 gpurun_out/sweep_traffic.log
