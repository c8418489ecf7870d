mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
for v in 0 2; do for h in 0 0.5 0.8; do echo "c2 v=$v h=$h $(PRGPU_HOT_FRAC=$h PRGPU_VARIANT=$v run c2)"; done; done
tail -n 30 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error|assert" | head
