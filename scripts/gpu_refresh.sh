# bench lines for every config at HEAD (profiles/r2_configs.md), the C5
# launch list and the ncu --set full capture of one C5 iteration's kernels
mkdir -p gpurun_out/r2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_c5.log 2>&1; echo "c5 rc=$?"
for c in c1 c2 c3 c4 c2series c5series c2k1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2/bench_$c.log 2>&1; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --config c2 --steps 5 --warmup 1 > gpurun_out/r2/ref_c2.log 2>&1; echo "ref c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
# one all-lanes iteration of C5 (host-driven launches: the second iteration's three kernels)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 3 -o gpurun_out/r2/c5_seg_full \
  python scripts/prof_pull.py --config c5 --launches 2 > gpurun_out/r2/c5_seg_full.log 2>&1; echo "ncu full rc=$?"
if [ -n "${REF_C5:-}" ]; then
  timeout 1500 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/r2/ref_c5.log 2>&1; echo "ref c5 rc=$?"
fi
