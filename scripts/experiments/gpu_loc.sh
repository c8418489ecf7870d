mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
echo "c3 locality $(run c3) | degree order $(PRGPU_LOCALITY=0 run c3)"
for m in 0 1 2 3; do echo "c3 locality K1MINB=$m $(PRGPU_K1MINB=$m run c3)"; done
echo "c3 locality nosplit $(PRGPU_K1SPLIT=0 run c3)"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
