run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
echo "c2 sb4 $(run c2) | sb8 $(PRGPU_LIB=build_alt/libprgpu_sb8.so run c2)"
echo "c2 sb4 $(run c2) | sb8 $(PRGPU_LIB=build_alt/libprgpu_sb8.so run c2)"
