run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c2 c2k1 c4; do for s in 0 6 5 3; do echo "$c skip=$s $(PRGPU_SKIP=$s run $c)"; done; done
sed -i 's/v5_c2/v6_c2/g; s/PRGPU_VARIANT=5/PRGPU_VARIANT=0/' scripts/gpu_ncu_v3.sh; bash scripts/gpu_ncu_v3.sh
