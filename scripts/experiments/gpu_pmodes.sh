timeout 900 python -m pytest tests/test_partition_gpu.py -x -q 2>&1 | tail -3
PRGPU_PART_MODES=0 timeout 900 python -m pytest tests/test_partition_gpu.py -x -q 2>&1 | tail -1
for m in 1 0; do
PRGPU_PART_MODES=$m PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e > gpurun_out/part.log 2>&1; echo "part modes=$m rc=$?"; grep "^{" gpurun_out/part.log | tail -1 | cut -c1-220
done
PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-e2e --config c5 > gpurun_out/part5.log 2>&1; echo "part c5 rc=$?"; grep "^{" gpurun_out/part5.log | tail -1 | cut -c1-220
