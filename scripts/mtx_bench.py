#!/usr/bin/env python3
"""Parallel MatrixMarket ingest vs the reference's parse (host only):
writes an RMAT-<scale> edge list as .mtx, then times prgpu_mtx_load (all
cores) and the reference's load_matrix_market (oracle/_ref), checks equality.
    python scripts/mtx_bench.py [scale] [dir]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2108_02997_b200 as prl  # noqa: E402
from pyoracle import Oracle, Ref  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
O = Oracle()
n, pairs = O.rmat(scale, 16, 0.57, 0.19, 0.19, 2108)
p = pairs.reshape(-1, 2).astype(np.int64) + 1
path = os.path.join(d, f"rmat{scale}.mtx")
with open(path, "w") as f:
    f.write("%%MatrixMarket matrix coordinate pattern general\n")
    f.write(f"{n} {n} {len(p)}\n")
    np.savetxt(f, p, fmt="%d")
size = os.path.getsize(path)
t = time.perf_counter()
el = prl.load_matrix_market(path)
t_nat = time.perf_counter() - t
t = time.perf_counter()
rn, rp = Ref().load_mtx(path)
t_ref = time.perf_counter() - t
assert rn == el.vertex_count and np.array_equal(rp, el.edges)
print(f"rmat{scale}.mtx {size / 1e6:.0f} MB, {len(p)} entries: native {t_nat:.3f} s "
      f"({size / t_nat / 1e9:.2f} GB/s, {os.cpu_count()} threads), reference {t_ref:.3f} s "
      f"({size / t_ref / 1e9:.3f} GB/s): {t_ref / t_nat:.1f}x")
os.remove(path)
