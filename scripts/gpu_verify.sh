# verification of HEAD: gpu tests, default bench, prof_pull per config
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
for c in c2 c2k1 c3 c4; do echo "$c $(run $c)"; done
tail -n 5 gpurun_out/pytest_gpu.log
tail -c 2500 gpurun_out/bench_full.log
