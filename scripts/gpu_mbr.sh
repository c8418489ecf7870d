./build_alt/mbr
for g in 32 64 128; do
echo "== ncu with granularity $g"
MBR_GRAN=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:gather -s 1 -c 1 --csv ./build_alt/mbr 2>&1 | grep -E '^"' | awk -F'","' '{print $(NF-2)" | "$NF}'
done
