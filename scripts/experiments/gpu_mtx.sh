mkdir -p gpurun_out
nproc
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/mtx_bench.py 22 /tmp 2>&1 | tail -1
PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/part.log 2>&1; echo "part rc=$?"; grep "^{" gpurun_out/part.log | tail -1 | cut -c1-600
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/ref.log | cut -c1-400
