run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c2 c2k1 c4; do echo "$c $(run $c) | unsorted $(PRGPU_ROW_SORT=0 run $c)"; done
PYTHONPATH=. PRGPU_TIMING_LOG=1 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -12
PYTHONPATH=. timeout 300 python scripts/e2e_probe.py 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 3
