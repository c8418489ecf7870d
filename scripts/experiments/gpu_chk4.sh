run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4 c5 c2; do echo "$c $(run $c)"; done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_c5_gpu.py -x -q -k "c4 or c5" 2>&1 | tail -2
