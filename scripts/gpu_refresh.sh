# round-1 evidence refresh: gpu tests, bench lines for every config, C2 launch lists + ncu of the
# widest kernels, the reference arm, and the partitioned (multi-GPU) path as one rank
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
bash scripts/gpu_bench_r1.sh
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "ref rc=$?"
for c in c2 c5; do
PRGPU_BENCH_PARTITION=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --config $c --no-e2e > gpurun_out/part_$c.log 2>&1; echo "part $c rc=$?"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
