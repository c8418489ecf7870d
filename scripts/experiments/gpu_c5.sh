mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem.txt; sleep 2; done ) &
MP=$!
PRGPU_TIMING_LOG=1 timeout 600 python scripts/prof_pull.py --config c5 --launches 4 > gpurun_out/c5_prof.log 2>&1; echo "c5 prof rc=$?"
tail -n 30 gpurun_out/c5_prof.log
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_bench.log 2>&1; echo "c5 bench rc=$?"
tail -c 2500 gpurun_out/c5_bench.log
kill $MP; sort -n gpurun_out/mem.txt | tail -1
P="python scripts/prof_pull.py --config c4 --launches 5"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/c4_pull $P > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
tail -3 gpurun_out/ncu_c4.log
