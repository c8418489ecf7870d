B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
PRGPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pull_kernel<.int.8, .int.2, .int.128" -s 4 -c 2 -o gpurun_out/r1_c2_pull $B > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
