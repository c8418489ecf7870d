mkdir -p gpurun_out
PRGPU_BENCH_PARTITION=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --config c5 > gpurun_out/part5.log 2>&1; echo "part c5 rc=$?"; grep "^{" gpurun_out/part5.log | tail -1 | cut -c1-1500
grep -v "^\[rank0\]:  \|^  " gpurun_out/part5.log | grep -i "error" | head -5
