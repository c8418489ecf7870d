M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for v in "" "PRGPU_SPLIT_MB=48"; do
  echo "== [$v]"
  env $v timeout 900 ncu -k regex:pull_kernel -c 8 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 2 2>&1 | grep -E '^"' | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}' | sed 's/(Params)//'
done
