run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
bq() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'GTEPS', round(d['ms_per_step'],3), 'ms/step')"; }
for b in 8 4; do for v in 0 5 6; do
  L=build_alt/libprgpu_pb$b.so
  echo "batch=$b minb=$v c2 $(PRGPU_LIB=$L PRGPU_K12P=$v run c2) | bench $(PRGPU_LIB=$L PRGPU_K12P=$v bq c2)"
done; done
