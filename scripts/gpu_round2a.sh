mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_c5.log
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c5.log 2>&1; echo "ref rc=$?"; tail -c 2000 gpurun_out/bench_ref_c5.log
