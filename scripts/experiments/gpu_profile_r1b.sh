mkdir -p gpurun_out
P="python scripts/prof_pull.py --launches 6"
for c in c2 c2k1 c4; do timeout 300 $P --config $c > gpurun_out/plain_$c.log 2>&1; done
timeout 200 $P --config c2k1 > gpurun_out/plainx.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/prof_c2k1 $P --config c2k1 > gpurun_out/ncu_c2k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/prof_c2 $P --config c2 > gpurun_out/ncu_c2.log 2>&1
cat gpurun_out/plain_*.log
