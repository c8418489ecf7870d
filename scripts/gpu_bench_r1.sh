# Round-1 evidence: bench line, launch list (host-loop mode), full ncu of the pull kernel.
mkdir -p gpurun_out
export PRGPU_VARIANT=${PRGPU_VARIANT:-0}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
PRGPU_NO_GRAPH=1 timeout 300 $B > gpurun_out/plain_ng.log 2>&1 && PRGPU_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 300 $B > gpurun_out/plain_g.log 2>&1 && timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/graphs_c2.csv $B > gpurun_out/ncu_graph.log 2>&1; echo "graph list rc=$?"
# the wide (all-lanes) kernel pair of the 3rd iteration: hub chunks, then packed + empty
PRGPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pull_kernel<.int.8, .int.2, .int.128" -s 4 -c 2 -o gpurun_out/r1_c2_pull $B > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -c 3000 gpurun_out/bench_full.log
