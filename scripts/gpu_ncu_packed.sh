mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:pull_kernel -s 5 -c 1 --clock-control none \
  -o gpurun_out/c5_packed_full python scripts/prof_pull.py --config c5 --launches 6 > gpurun_out/c5_packed_full.log 2>&1; echo "full rc=$?"
