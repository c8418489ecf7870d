#!/usr/bin/env bash
# the segmented hub pull: parity tests, then A/B runs (scripts/seg_ab.py)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_seg_gpu.py -m gpu -q -x > gpurun_out/seg_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/seg_pytest.log
for c in ${CONFIGS:-c2 c5}; do
    PRGPU_TIMING_LOG=${TLOG:-} timeout 1500 python scripts/seg_ab.py $c ${STEPS:-5} "$@" 2>&1 | grep -v "^\[session\]\|^\[results\]" | tee gpurun_out/seg_ab_$c.log
done
