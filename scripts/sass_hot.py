#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]; body = rows[1:]
si = h.index('Warp Stall Sampling (All Samples)'); src = h.index('Source'); ad = h.index('Address')
stall_cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
tot = sum(float(r[si] or 0) for r in body)
print('total samples', tot)
for idx, r in sorted(enumerate(body), key=lambda x: -float(x[1][si] or 0))[:top]:
    st = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{idx:5d} {float(r[si])/tot*100:5.1f}% {r[src].strip()[:60]:60s} {st[0][1]}={int(st[0][0])} {st[1][1]}={int(st[1][0])}")
