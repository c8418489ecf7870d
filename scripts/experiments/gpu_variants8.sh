mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 4 5 6; do PRGPU_VARIANT=$v timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_v$v.log').read().strip().splitlines()[-1]); print('bench c2 v=$v', round(d['value'],1), 'GTEPS', round(d['ms_per_step'],2), 'ms/step, pull', round(d['roofline']['per_launch_ms'],3), 'ms frac', round(d['roofline']['frac'],3))"; done
for v in 5 6; do PRGPU_VARIANT=$v python -m pytest tests/test_parity_gpu.py -x -q -k "c2 or batched" 2>&1 | tail -n 1; done
tail -n 40 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error|assert" | head
