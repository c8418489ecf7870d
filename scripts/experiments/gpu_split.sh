run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c2 c2k1 c3 c4; do echo "$c split $(run $c) | nosplit $(PRGPU_SPLIT=0 run $c)"; done
for s in 6 5; do echo "c2 skip=$s $(PRGPU_SKIP=$s run c2)"; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 3
