mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
for m in 0 1 2; do echo "c2 L2MODE=$m $(PRGPU_L2MODE=$m run c2)"; done
for v in 2 3; do echo "c2 v=$v $(PRGPU_VARIANT=$v run c2)"; done
for m in 0 1 2; do echo "c2k1 L2MODE=$m $(PRGPU_L2MODE=$m run c2k1)"; done
for m in 0 1; do echo "c4 L2MODE=$m $(PRGPU_L2MODE=$m run c4)"; done
for m in 0 1; do echo "c3 L2MODE=$m $(PRGPU_L2MODE=$m PRGPU_VARIANT=1 run c3)"; done
tail -n 40 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error|assert" | head
