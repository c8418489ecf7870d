run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4; do echo "$c nq2 $(run $c) | nq4 $(PRGPU_K1NQ=4 run $c)"; done
echo "c2k1 split nq2 $(PRGPU_K1SPLIT=1 run c2k1) | nq4 $(PRGPU_K1SPLIT=1 PRGPU_K1NQ=4 run c2k1)"
