run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
PRGPU_TIMING_LOG=1 timeout 300 python scripts/prof_pull.py --config c2 --all 2>&1 | grep "^launch" | tr '\n' ' '; echo
PRGPU_MODES=0 PRGPU_TIMING_LOG=1 timeout 300 python scripts/prof_pull.py --config c2 --all 2>&1 | grep "^launch" | tr '\n' ' '; echo
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 3
