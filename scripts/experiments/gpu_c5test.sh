mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_c5_gpu.py tests/test_parity_gpu.py -k "c5 or graph_rows" -x -q -s > gpurun_out/c5_test.log 2>&1; echo "rc=$?"
tail -n 30 gpurun_out/c5_test.log
free -g | head -2
