mkdir -p gpurun_out
P="python scripts/prof_pull.py --config c5 --launches 4"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 2 -c 1 -o gpurun_out/c5_pull $P > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
tail -3 gpurun_out/ncu_c5.log
