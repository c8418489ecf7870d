run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c3 c4 c2k1 c1 c2; do echo "$c $(run $c) | minb3-packed $(PRGPU_K1MINB=0 run $c)"; done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
