timeout 900 python -m pytest tests/test_partition_gpu.py -x -q 2>&1 | tail -3
PRGPU_DEAL=0 timeout 900 python -m pytest tests/test_partition_gpu.py -x -q 2>&1 | tail -1
timeout 900 python scripts/exchange_volume.py c2 2>&1 | tail -4
for m in 1 0; do
PRGPU_DEAL=$m PRGPU_BENCH_PARTITION=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e > gpurun_out/part.log 2>&1; echo "part deal=$m rc=$?"; grep "^{" gpurun_out/part.log | tail -1 | cut -c1-200
done
timeout 1200 python -m pytest tests/test_c5_gpu.py -x -q -k two_rank 2>&1 | tail -2
