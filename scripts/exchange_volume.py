#!/usr/bin/env python3
"""Fused-exchange volume of the partitioned solve at N ranks, measured by
emulating the N ranks on one GPU (distributed.emulate, fused=True): bytes each
rank stores into its peers per all-lanes iteration (max over ranks), with the
needed-only mask and without it (PRGPU_NEED=0).
    python scripts/exchange_volume.py [config] [ranks,...] [need modes: 1,0]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2108_02997_b200 as prl  # noqa: E402
from paper_2108_02997_b200 import distributed  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
ranks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 8]
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "0"]
g = prl.generate_rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, bench.SEED)
out = {"workload": cfg["workload"], "ranks": {}}
for n in ranks:
    row = {}
    for need in modes:
        os.environ["PRGPU_NEED"] = need
        r = distributed.emulate(g, cfg["alphas"], n, cfg["tol"], prl.NormKind(cfg["norm"]), 500, want_ranks=False,
                                fused=True)
        row["needed_only" if need == "1" else "every_peer"] = r.sent_bytes
    out["ranks"][n] = row
    print(n, row, flush=True)
print(json.dumps(out))
