run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for ch in 2048 4096 8192 16384; do echo "c4 chunk=$ch $(PRGPU_CHUNK=$ch run c4)"; done
for ch in 1024 2048 4096 8192; do echo "c5 chunk=$ch $(PRGPU_CHUNK=$ch run c5)"; done
for ch in 1024 2048 4096; do echo "c2 chunk=$ch $(PRGPU_CHUNK=$ch run c2)"; done
