#!/usr/bin/env python3
"""Profiling driver: builds a bench config's graph and runs the pull kernel as
plain launches (no CUDA graph), so ncu can see each launch.

    python scripts/prof_pull.py --config c2 --launches 8
    ncu --set full -k regex:pull_kernel -s 4 -c 1 python scripts/prof_pull.py ...
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2108_02997_b200 as prl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(bench.CONFIGS))
    ap.add_argument("--launches", type=int, default=8)
    ap.add_argument("--all", action="store_true", help="run to convergence")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    if cfg["kind"] == "rmat":
        g = prl.generate_rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, bench.SEED)
    else:
        g = prl.generate_grid(cfg["side"], 0.6, 0.01, bench.SEED)
    s = prl.Session(g, cfg["alphas"], cfg["tol"], prl.NormKind(cfg["norm"]), 500,
                    cfg.get("stop_mask", 0))
    ms = s.time_pull(500 if args.all else args.launches)
    info = g.info
    print(f"{args.config}: N={g.vertex_count} E={g.edge_count()} hub={info.hub_rows} "
          f"warp={info.warp_rows} thread={info.thread_rows} empty={info.empty_rows} "
          f"pull {ms:.4f} ms/launch")


if __name__ == "__main__":
    main()
