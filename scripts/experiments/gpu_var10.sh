run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for v in 0 2; do echo "c2 v=$v $(PRGPU_VARIANT=$v run c2)"; done
for ch in 1024 4096; do echo "c2 chunk=$ch $(PRGPU_CHUNK=$ch run c2)"; done
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print('bench c2', round(d['value'],1), 'GTEPS', round(d['ms_per_step'],2), 'ms/step, pull', round(d['roofline']['per_launch_ms'],3), 'ms frac', round(d['roofline']['frac'],3))"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1
