run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4 c5; do echo "$c slr $(run $c) | off $(PRGPU_SLR=0 run $c)"; done
for mb in 16 48; do echo "c5 slr ${mb}MB $(PRGPU_SLR_MB=$mb run c5)"; done
for d in 256 4096; do echo "c5 slr deg>$d $(PRGPU_SLR_DEG=$d run c5)"; done
timeout 900 python -m pytest tests/test_c5_gpu.py tests/test_parity_gpu.py -x -q -k "c4 or c5 or batched" 2>&1 | tail -3
