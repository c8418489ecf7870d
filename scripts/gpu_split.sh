mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "split" 2>&1 | tail -3
export LAUNCHES=6
bash scripts/gpu_ab.sh c5 "" "PRGPU_SPLIT_MB=16" "PRGPU_SPLIT_MB=32" "PRGPU_SPLIT_MB=48" "PRGPU_SPLIT_MB=64" "PRGPU_SPLIT_MB=96" "PRGPU_SPLIT_MB=48 PRGPU_GPOL=1 PRGPU_HOT_MB=48" ""
export LAUNCHES=8
bash scripts/gpu_ab.sh c4 "" "PRGPU_SPLIT_MB=16" "PRGPU_SPLIT_MB=32" "PRGPU_SPLIT_MB=48" "PRGPU_SPLIT_MB=64" ""
bash scripts/gpu_ab.sh c2 "" "PRGPU_SPLIT_MB=16" "PRGPU_SPLIT_MB=32" "PRGPU_SPLIT_MB=48" "PRGPU_SPLIT_MB=64" ""
