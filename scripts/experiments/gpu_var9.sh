run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for v in 0 1 2 3; do echo "c2 v=$v $(PRGPU_VARIANT=$v run c2)"; done
for v in 0 2; do for c in c2k1 c3 c4; do echo "$c v=$v $(PRGPU_VARIANT=$v run $c)"; done; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1
