run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for L in build_alt/libprgpu_head.so build_alt/libprgpu_nobcast.so paper_2108_02997_b200/libprgpu.so; do
  for s in 0 6 5; do echo "$L c2 skip=$s $(PRGPU_LIB=$L PRGPU_SKIP=$s run c2)"; done
done
for L in build_alt/libprgpu_nobcast.so paper_2108_02997_b200/libprgpu.so; do
  for v in 1 2 3; do echo "$L c2 var=$v $(PRGPU_LIB=$L PRGPU_VARIANT=$v run c2)"; done
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 3
