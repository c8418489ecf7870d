run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for L in paper_2108_02997_b200/libprgpu.so build_alt/libprgpu_coal.so; do
  echo "$L c4 $(PRGPU_LIB=$L run c4) | c2k1 $(PRGPU_LIB=$L run c2k1) | c2 $(PRGPU_LIB=$L run c2)"
done
PRGPU_LIB=build_alt/libprgpu_coal.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1 or c4 or known or batched" 2>&1 | tail -2
