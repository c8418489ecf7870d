run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4 c2k1 c2 c5; do echo "$c row-order $(run $c) | out-degree order $(PRGPU_SRC_ORDER=2 run $c)"; done
PRGPU_SRC_ORDER=2 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1 or c2 or batched" 2>&1 | tail -2
