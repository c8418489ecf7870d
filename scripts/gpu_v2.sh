run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for v in 0 1 2 3 4; do echo "c2 var2=$v $(PRGPU_VARIANT2=$v run c2) skip5 $(PRGPU_SKIP=5 PRGPU_VARIANT2=$v run c2)"; done
