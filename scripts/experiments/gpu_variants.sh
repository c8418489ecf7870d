mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1 2 3 4; do PRGPU_VARIANT=$v timeout 120 python scripts/prof_pull.py --config c2k1 --launches 10 > gpurun_out/var_c2k1_$v.log 2>&1; done
for v in 0 1 2; do PRGPU_VARIANT=$v timeout 120 python scripts/prof_pull.py --config c2 --launches 10 > gpurun_out/var_c2_$v.log 2>&1; done
for v in 0 1 2 4; do PRGPU_VARIANT=$v timeout 300 python scripts/prof_pull.py --config c4 --launches 6 > gpurun_out/var_c4_$v.log 2>&1; done
for v in 0 1 4; do PRGPU_VARIANT=$v timeout 120 python scripts/prof_pull.py --config c3 --launches 10 > gpurun_out/var_c3_$v.log 2>&1; done
tail -n 3 gpurun_out/pytest_gpu.log; for f in gpurun_out/var_*.log; do echo "$f: $(tail -n 1 $f)"; done
