mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gpu.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
echo "c5 nosplit $(PRGPU_SPLIT=0 run c5)"
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench c2 rc=$?"
P="python scripts/prof_pull.py --config c5 --launches 3"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pull_kernel<.int.4, .int.1," -s 2 -c 2 -o gpurun_out/c5_pull2 $P > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
tail -2 gpurun_out/ncu_c5.log
