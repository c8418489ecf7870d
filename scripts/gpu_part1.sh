export PRGPU_BENCH_PARTITION=1
python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --config c2 --steps 3 --warmup 3 2>&1 | grep '^{' | cut -c1-600
python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --config c2 --steps 3 --warmup 3 --shard 2>&1 | grep '^{' | cut -c1-600
python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --config c5 --steps 3 --warmup 3 2>&1 | tail -3 | cut -c1-900
