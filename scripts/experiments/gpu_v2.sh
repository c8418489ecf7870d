run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
echo "base c2 $(run c2) skip5 $(PRGPU_SKIP=5 run c2)"
echo "async c2 $(PRGPU_LIB=build_alt/libprgpu_async.so run c2) skip5 $(PRGPU_LIB=build_alt/libprgpu_async.so PRGPU_SKIP=5 run c2)"
