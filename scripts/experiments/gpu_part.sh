export PRGPU_BENCH_PARTITION=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/part.log 2>&1; echo rc=$?
grep "^{" gpurun_out/part.log | tail -1 | cut -c1-2500; tail -3 gpurun_out/part.log | cut -c1-300
