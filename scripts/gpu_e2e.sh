run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for L in build_alt/libprgpu_head.so build_alt/libprgpu_nobcast.so paper_2108_02997_b200/libprgpu.so; do
  for s in 0 6; do echo "$L c2 skip=$s $(PRGPU_LIB=$L PRGPU_SKIP=$s run c2)"; done
done
PYTHONPATH=. timeout 300 python scripts/e2e_probe.py 2>&1 | tail -4
PRGPU_TIMING_LOG=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -v "^launch" | tail -12
