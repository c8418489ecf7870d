#!/usr/bin/env bash
# A/B runner for the tuning switches, run on the
# GPU box from the repo root:
#   gpurun -- 'bash scripts/gpu_ab.sh c5 "" "PRGPU_CHUNK=512" "PRGPU_SPLIT=0"'
# Each variant is a space-separated list of VAR=value settings ("" = the
# defaults); every variant times LAUNCHES pull launches with
# scripts/prof_pull.py on CONFIG and prints one line per variant.
#   NCU=regex  additionally captures `ncu --set full` of the first matching
#              kernel for the first variant into gpurun_out/ab_<config>.ncu-rep
set -u
cfg=${1:?config}; shift
launches=${LAUNCHES:-6}
mkdir -p gpurun_out
for v in "$@"; do
    line=$(env $v timeout 600 python scripts/prof_pull.py --config "$cfg" --launches "$launches" 2>&1 | tail -n 1)
    echo "$cfg [${v:-defaults}] $line"
done
if [ -n "${NCU:-}" ]; then
    env ${1:-} timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$NCU" -s 2 -c 1 \
        -o "gpurun_out/ab_$cfg" python scripts/prof_pull.py --config "$cfg" --launches 4 \
        > "gpurun_out/ab_ncu_$cfg.log" 2>&1
    echo "ncu rc=$? -> gpurun_out/ab_$cfg.ncu-rep"
fi
