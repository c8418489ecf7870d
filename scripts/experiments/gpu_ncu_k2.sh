mkdir -p gpurun_out
P="python scripts/prof_pull.py --config c2 --launches 6"
export PRGPU_LIB=build_alt/prof.so PRGPU_NO_GRAPH=1
timeout 200 $P > gpurun_out/p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 7 -c 1 -o gpurun_out/k2b_c2 $P > gpurun_out/n.log 2>&1; echo "rc=$?"
