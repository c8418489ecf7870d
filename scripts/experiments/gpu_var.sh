run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for v in 0 1 2 3; do echo "c2 var=$v $(PRGPU_VARIANT=$v run c2)"; done
for v in 0 1 2 3; do echo "c2k1 var=$v $(PRGPU_VARIANT=$v run c2k1)"; done
