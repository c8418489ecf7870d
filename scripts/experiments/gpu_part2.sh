mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partition_gpu.py -x -q > gpurun_out/pt.log 2>&1; echo "part tests rc=$?"; tail -n 5 gpurun_out/pt.log
for ex in peer nccl; do
PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --exchange $ex > gpurun_out/part.log 2>&1; echo "part $ex rc=$?"; grep "^{" gpurun_out/part.log | tail -1 | cut -c1-300
done
PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --config c5 > gpurun_out/part5.log 2>&1; echo "part c5 rc=$?"; grep "^{" gpurun_out/part5.log | tail -1 | cut -c1-300
