export LAUNCHES=6
bash scripts/gpu_ab.sh c5 "" "PRGPU_PERSIST_MB=16" "PRGPU_PERSIST_MB=32" "PRGPU_PERSIST_MB=54" "PRGPU_PERSIST_MB=80" \
  "PRGPU_GPOL=4 PRGPU_HOT_MB=54" "PRGPU_GPOL=5 PRGPU_HOT_MB=54" "PRGPU_GPOL=4 PRGPU_HOT_MB=16" \
  "PRGPU_PERSIST_MB=54 PRGPU_GPOL=5 PRGPU_HOT_MB=54" ""
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed
for v in "PRGPU_PERSIST_MB=54" "PRGPU_GPOL=4 PRGPU_HOT_MB=54" "PRGPU_GPOL=5 PRGPU_HOT_MB=54"; do
  echo "== [$v] hub launch"
  env $v timeout 900 ncu -k regex:pull_kernel -s 4 -c 1 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 6 2>&1 | grep -E '^"' | awk -F'","' '{print $(NF-2)" | "$NF}'
done
