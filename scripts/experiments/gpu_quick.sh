# quick perf + parity check: per-launch pull time on the probe configs, C2 bench, gpu tests
mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in ${CONFIGS:-c2s20 c2 c2k1 c3 c4}; do echo "$(run $c)"; done
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print('bench c2', round(d['value'],1), 'GTEPS', round(d['ms_per_step'],2), 'ms/step, pull', round(d['roofline']['per_launch_ms'],3), 'ms frac', round(d['roofline']['frac'],3))"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2
