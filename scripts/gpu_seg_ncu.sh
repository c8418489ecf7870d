#!/usr/bin/env bash
# per-kernel time / DRAM bytes / L2 hit rate of an iteration's pull kernels
# (host-driven launches): bash scripts/gpu_seg_ncu.sh c5 tag "VAR=v ..."
set -u
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out
env $* timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum \
    --clock-control none -k regex:pull_kernel --csv --log-file gpurun_out/seg_ncu_${cfg}_${tag}.csv \
    python scripts/prof_pull.py --config $cfg --launches ${LAUNCHES:-2} > gpurun_out/seg_ncu_${cfg}_${tag}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/seg_ncu_${cfg}_${tag}.log
python - <<PY
import csv
rows=list(csv.reader(l for l in open("gpurun_out/seg_ncu_${cfg}_${tag}.csv") if l.startswith('"')))
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
d={}
for r in rows[1:]:
    d.setdefault((r[ii],r[ki]),{})[r[mi]]=float(r[vi].replace(',',''))
for (i,k),m in d.items():
    t=m.get("gpu__time_duration.sum",0)/1e6
    if t<0.05: continue
    print(i,k[:60],"%.2f ms"%t,"dramR %.1f GB"%(m.get("dram__bytes_read.sum",0)/1e9),"dramW %.1f GB"%(m.get("dram__bytes_write.sum",0)/1e9),"L2hit %.1f%%"%m.get("lts__t_sector_hit_rate.pct",0),"L2 read sectors %.2f G"%(m.get("lts__t_sectors_op_read.sum",0)/1e9))
PY
