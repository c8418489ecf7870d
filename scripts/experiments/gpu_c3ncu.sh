mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
P="python scripts/prof_pull.py --config c3 --launches 4"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 2 -c 2 -o gpurun_out/c3_pull $P > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"; tail -1 gpurun_out/ncu_c3.log
