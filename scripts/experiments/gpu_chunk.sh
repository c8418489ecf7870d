run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c2 c2k1 c4; do for ch in 2048 4096 16384; do echo "$c chunk=$ch $(PRGPU_CHUNK=$ch run $c)"; done; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1
