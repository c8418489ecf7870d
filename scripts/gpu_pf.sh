export LAUNCHES=6
bash scripts/gpu_ab.sh c5 "" "PRGPU_PF=1" "PRGPU_PF=1 PRGPU_GPOL=1 PRGPU_HOT_MB=64" "PRGPU_PF=1 PRGPU_GPOL=1 PRGPU_HOT_MB=32" "PRGPU_PF=1 PRGPU_CHUNK=1024" "PRGPU_PF=1 PRGPU_CHUNK=4096" ""
bash scripts/gpu_ab.sh c2 "" "PRGPU_PF=1" ""
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct
for v in "PRGPU_PF=1" "PRGPU_PF=1 PRGPU_GPOL=1 PRGPU_HOT_MB=64"; do
  for s in 4 5; do
  echo "== [$v] launch $s"
  env $v timeout 900 ncu -k regex:pull_kernel -s $s -c 1 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 6 2>&1 | grep -E '^"' | awk -F'","' '{print $(NF-2)" | "$NF}'
  done
done
