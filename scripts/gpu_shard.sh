timeout 1500 python -m pytest tests/test_shard_gpu.py tests/test_multiproc_gpu.py tests/test_partition_gpu.py -q -s 2>&1 | grep -v "^$" | tail -8
