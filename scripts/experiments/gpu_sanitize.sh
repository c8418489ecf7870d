export PRGPU_NO_GRAPH=1
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -5 gpurun_out/memcheck_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_parity_gpu.py -x -q -k "known or structural or batched_lane_modes" > gpurun_out/memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -5 gpurun_out/memcheck_tests.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_partition_gpu.py -x -q -k "fused" > gpurun_out/memcheck_part.log 2>&1; echo "memcheck part rc=$?"; tail -5 gpurun_out/memcheck_part.log
