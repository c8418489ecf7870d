timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for c in "c5 5"; do
python scripts/loop_ab.py $c
PRGPU_LIB=build_alt/libprgpu_r2a.so python scripts/loop_ab.py $c
done
python scripts/loop_ab.py c5series 3 2>/dev/null | tail -1
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct
timeout 900 ncu -k regex:pull_kernel -s 4 -c 2 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 4 2>&1 | grep -E '^"' | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}'
