mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
for v in 0 2 4; do echo "c2 v=$v $(PRGPU_VARIANT=$v run c2)"; done
for v in 0 4; do PRGPU_VARIANT=$v timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_v$v.log').read().strip().splitlines()[-1]); print('bench c2 v=$v', round(d['value'],1), 'GTEPS', round(d['ms_per_step'],2), 'ms/step frac', round(d['roofline']['frac'],3))"; done
tail -n 40 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error|assert" | head
