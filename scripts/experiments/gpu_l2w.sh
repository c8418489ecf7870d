run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
echo "base $(run c2)"
echo "mode5 $(PRGPU_L2MODE=5 run c2)"
for mb in 16 32 48 64 96; do
 for m in 3 4; do echo "mode$m hot=$mb $(PRGPU_L2MODE=$m PRGPU_HOT_MB=$mb run c2)"; done
done
for mb in 8 16 32; do echo "k1 mode3 hot=$mb $(PRGPU_L2MODE=3 PRGPU_HOT_MB=$mb run c2k1)"; done
echo "k1 base $(run c2k1)"
