mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4 c3 c2k1 c1; do
 echo "$c base $(run $c) | split $(PRGPU_K1SPLIT=1 run $c) | hub4 $(PRGPU_K1SPLIT=1 PRGPU_K1MINB=1 run $c) | packed4 $(PRGPU_K1SPLIT=1 PRGPU_K1MINB=2 run $c) | both4 $(PRGPU_K1SPLIT=1 PRGPU_K1MINB=3 run $c)"
done
