set -x; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1
timeout 200 python bench.py --config c2k1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2k1.log 2>&1
timeout 200 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 200 $B --config c2 > gpurun_out/plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B --config c2 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 40 -c 1 -o gpurun_out/prof_c2 $B --config c2 > gpurun_out/ncu2.log 2>&1
timeout 200 $B --config c2k1 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 40 -c 1 -o gpurun_out/prof_c2k1 $B --config c2k1 > gpurun_out/ncu3.log 2>&1
for f in gpurun_out/*.log; do echo == $f; tail -n 3 $f | cut -c1-600; done
