mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c3 c2k1 c4 c1; do echo "$c $(run $c)"; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
