# C5 hub-chunk kernel under ncu: defaults vs gather policies (DRAM bytes, L2 hits, time)
mkdir -p gpurun_out
K='regex:pull_kernel'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for v in "" "PRGPU_GPOL=1 PRGPU_HOT_MB=64" "PRGPU_GPOL=1 PRGPU_HOT_MB=16" "PRGPU_L2MODE=2"; do
  echo "== [$v]"
  env $v timeout 900 ncu -k "$K" -s 4 -c 1 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 6 2>&1 | grep -E '^"' | awk -F'","' '{print $(NF-3)" | "$(NF-2)" | "$NF}'
done
timeout 900 ncu --set full --import-source on -k "$K" -s 4 -c 1 --clock-control none \
  -o gpurun_out/c5_hub_full python scripts/prof_pull.py --config c5 --launches 6 > gpurun_out/c5_hub_full.log 2>&1; echo "full rc=$?"
