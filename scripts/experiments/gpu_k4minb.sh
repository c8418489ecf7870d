run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for r in 1 2; do for v in 0 5 7 8; do echo "c5 k4cfg=$v $(PRGPU_K4CFG=$v run c5)"; done; done
bq() { timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'GTEPS', round(d['ms_per_step'],3), 'ms/step')"; }
for v in 0 7; do echo "c5 bench k4cfg=$v $(PRGPU_K4CFG=$v bq c5)"; echo "c2 bench k4cfg=$v $(PRGPU_K4CFG=$v bq c2)"; done
