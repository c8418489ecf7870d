run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
bq() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'GTEPS', round(d['ms_per_step'],3), 'ms/step')"; }
for L in paper_2108_02997_b200/libprgpu.so build_alt/libprgpu_pair.so; do
  echo "$L c2 $(PRGPU_LIB=$L run c2) | bench $(PRGPU_LIB=$L bq c2) | c5 $(PRGPU_LIB=$L run c5)"
done
PRGPU_LIB=build_alt/libprgpu_pair.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "batched or c2 or c1_det" 2>&1 | tail -2
