PRGPU_LIB=build_alt/libprgpu_sw.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
python scripts/loop_ab.py c5 5
PRGPU_LIB=build_alt/libprgpu_sw.so python scripts/loop_ab.py c5 5
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
PRGPU_LIB=build_alt/libprgpu_sw.so timeout 900 ncu -k regex:pull_kernel -s 4 -c 2 --metrics $M --clock-control none --csv \
     python scripts/prof_pull.py --config c5 --launches 4 2>&1 | grep -E '^"' | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}'
