set -x
for v in 0 4 6; do
  echo "variant $v" >> gpurun_out/probe_timing.txt
  WSVD_ATTN_VARIANT=$v timeout 120 python tools/timing.py --reps 20 >> gpurun_out/probe_timing.txt 2>&1
done
for v in 0 4; do
  WSVD_ATTN_VARIANT=$v timeout 300 ncu -k regex:decode_attn -c 2 --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__issue_active.avg.pct_of_peak_sustained_active --csv python tools/timing.py --reps 2 > gpurun_out/probe_ncu_$v.csv 2>&1
done
