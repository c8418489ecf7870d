mkdir -p gpurun_out
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 6 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for v in 0 1 2 3 4 5; do echo "c5 k4cfg=$v $(PRGPU_K4CFG=$v run c5)"; done
echo "c5 nosplit $(PRGPU_SPLIT=0 run c5)"
for v in 0 1 3; do echo "c2s20-like c5-small? skip"; done 2>/dev/null | head -0
P="python scripts/prof_pull.py --config c5 --launches 3"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pull_kernel<2, 2" -s 2 -c 2 -o gpurun_out/c5_pull2 $P > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
tail -2 gpurun_out/ncu_c5.log
