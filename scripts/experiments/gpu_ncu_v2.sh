mkdir -p gpurun_out
P="python scripts/prof_pull.py --launches 5"
export PRGPU_VARIANT=1
timeout 200 $P --config c2k1 > gpurun_out/p1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/v2_c2k1 $P --config c2k1 > gpurun_out/n1.log 2>&1
timeout 300 $P --config c4 > gpurun_out/p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/v2_c4 $P --config c4 > gpurun_out/n2.log 2>&1
export PRGPU_VARIANT=2
timeout 200 $P --config c2 > gpurun_out/p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/v2_c2 $P --config c2 > gpurun_out/n3.log 2>&1
tail -n 2 gpurun_out/n*.log
