mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
for v in 0 1 3; do for h in 0 0.5; do echo "c2k1 v=$v hot=$h $(PRGPU_VARIANT=$v PRGPU_HOT_FRAC=$h run c2k1)"; done; done
for v in 1; do for h in 0 0.3 0.5 0.7; do echo "c4 v=$v hot=$h $(PRGPU_VARIANT=$v PRGPU_HOT_FRAC=$h run c4)"; done; done
for v in 0 1; do for h in 0 0.5; do echo "c3 v=$v hot=$h $(PRGPU_VARIANT=$v PRGPU_HOT_FRAC=$h run c3)"; done; done
for v in 0 2; do for h in 0 0.5; do echo "c2 v=$v hot=$h $(PRGPU_VARIANT=$v PRGPU_HOT_FRAC=$h run c2)"; done; done
tail -n 2 gpurun_out/pytest_gpu.log
