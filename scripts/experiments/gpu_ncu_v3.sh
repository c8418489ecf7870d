mkdir -p gpurun_out
P="python scripts/prof_pull.py --launches 5"
export PRGPU_VARIANT=5; timeout 200 $P --config c2 > gpurun_out/p3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/v5_c2 $P --config c2 > gpurun_out/n3.log 2>&1
tail -n 2 gpurun_out/n3.log
