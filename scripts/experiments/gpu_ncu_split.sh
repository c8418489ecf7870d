mkdir -p gpurun_out
P="python scripts/prof_pull.py --config c2 --launches 6"
PRGPU_NO_GRAPH=1 timeout 200 $P > gpurun_out/p.log 2>&1 && PRGPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 6 -c 2 -o gpurun_out/split_c2 $P > gpurun_out/n.log 2>&1; echo "rc=$?"
