mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_c5_gpu.py tests/test_parity_gpu.py -k "c5 or graph_rows" -x -q > gpurun_out/c5_test.log 2>&1; echo "c5 test rc=$?"; tail -n 3 gpurun_out/c5_test.log
run() { timeout 300 python scripts/prof_pull.py --config $1 --launches 8 2>&1 | tail -n 1 | sed 's/N=[0-9]* E=[0-9]* hub=[0-9]* warp=[0-9]* thread=[0-9]* empty=[0-9]*//'; }
for c in c4 c2k1 c2 c5; do for kb in off 32 64 96 128 192; do
  if [ $kb = off ]; then echo "$c l1hot=off $(run $c)"; else echo "$c l1hot=$kb $(PRGPU_L1HOT_KB=$kb run $c)"; fi
done; done
