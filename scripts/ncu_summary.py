#!/usr/bin/env python3
"""Summarise an ncu report (raw page) into the numbers DESIGN.md/profiles cite."""
import csv, subprocess, sys, json
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'sm__cycles_active.avg', 'gpc__cycles_elapsed.max', 'smsp__inst_executed.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed']
def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row)); u = dict(zip(h, units))
        item = {'kernel': d.get('Kernel Name', '')[:80]}
        for k in KEYS:
            if k in d:
                item[k] = d[k] + (' ' + u[k] if u.get(k) else '')
        stalls = sorted(((float(d[k].replace(',', '') or 0), k) for k in h
                         if 'pcsamp_warps_issue_stalled' in k and 'not_issued' not in k), reverse=True)[:5]
        item['top_stalls'] = [f"{k.split('stalled_')[1]}={int(v)}" for v, k in stalls]
        res.append(item)
    return res
if __name__ == '__main__':
    for p in sys.argv[1:]:
        for it in summary(p):
            print(p); print(json.dumps(it, indent=1))
