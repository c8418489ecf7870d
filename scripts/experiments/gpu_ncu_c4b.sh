P="python scripts/prof_pull.py --config c4 --launches 4"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 2 -c 2 -o gpurun_out/c4_split $P > gpurun_out/ncu_c4b.log 2>&1; echo "ncu rc=$?"
