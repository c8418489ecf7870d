run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1; }
export PRGPU_VARIANT=2
for c in c2 c2k1; do for s in 0 1 2 4 3 5 6 7; do echo "$c skip=$s $(PRGPU_SKIP=$s run $c)"; done; done
