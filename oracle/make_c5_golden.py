#!/usr/bin/env python3
"""Writes tests/golden/c5_rmat28.{json,npz} from a run of the REFERENCE'S OWN
pagerank() (pagerank.hpp:70-108) on BASELINE.json configs[4]: RMAT-28
(268,435,456 vertices), alphas {.95, .85, .75}, tau 1e-6, L2, max 500.

TEST INFRASTRUCTURE ONLY.  Run here (needs /root/reference, ~35 GB of RAM and
hours of CPU):

    make -C oracle c5
    python oracle/make_c5_golden.py run        # C2/C4 fingerprint pins, then the scale-28 run
    python oracle/make_c5_golden.py summarize  # -> tests/golden/c5_rmat28.*

`run` first builds RMAT-22 and RMAT-26 with the same in-place builder
(oracle/csr_inplace.hpp) and requires their fingerprints to equal the C2 / C4
goldens, which the reference's own build_csr wrote (make_goldens.py); then
c5_golden builds RMAT-28 and runs the three lanes (one thread each).  The
full rank vectors stay in oracle/_c5/ (6.4 GB, never committed or shipped);
the golden keeps what a GPU test can compare at full size:
  * per lane: iterations, converged, the err trace (every iteration's L2
    norm of the rank change), the reference's loop time;
  * ranks at 65,536 seeded sample vertices and at the top-4096 ranks;
  * Sum(ranks) in long double; 8 seeded random-sign projections Sum(w_i r_i);
  * per 2^16-vertex block: the sum (long double) and the maximum.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")
WORK = os.path.join(HERE, "_c5")
BIN = os.path.join(HERE, "_ref", "c5_golden")
ALPHAS = [0.95, 0.85, 0.75]
N = 1 << 28
BLOCK = 1 << 16


def pin(scale, golden):
    out = os.path.join(WORK, f"s{scale}")
    os.makedirs(out, exist_ok=True)
    subprocess.run([BIN, str(scale), out, "--check"], check=True)
    got = json.load(open(os.path.join(out, "fingerprint.json")))
    want = json.load(open(os.path.join(GOLD, golden)))["graph"]
    for k, v in got.items():
        if want[k] != v:
            raise SystemExit(f"scale {scale}: {k} {v} != reference {want[k]}")
    print(f"scale {scale}: fingerprint equals the reference build_csr's ({golden})")


def run():
    subprocess.run(["make", "-s", "-C", HERE, "c5"], check=True)
    pin(22, "c2_rmat22.json")
    pin(26, "c4_rmat26.json")
    out = os.path.join(WORK, "s28")
    os.makedirs(out, exist_ok=True)
    subprocess.run([BIN, "28", out, "--norm", "l2", "--tol", "1e-6", "--max-iter", "500",
                    *map(str, ALPHAS)], check=True)


def sample_idx(n, k=65536):
    rs = np.random.default_rng(20210806)
    return np.sort(rs.choice(n, size=k, replace=False)).astype(np.int64)


def projections(r, count=8, seed=2108):
    """Sum w_i r_i for seeded w_i in {-1, +1} (counter-based: w depends on i only)."""
    out = []
    i = np.arange(r.size, dtype=np.uint64)
    for j in range(count):
        z = (i + np.uint64(j + 1) * np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        w = np.where((z >> np.uint64(63)) == 1, -1.0, 1.0)
        out.append(float(np.sum((w * r).astype(np.longdouble))))
        del z, w
    return out


def summarize():
    fp = json.load(open(os.path.join(WORK, "s28", "fingerprint.json")))
    idx = sample_idx(N)
    arrays = dict(sample_idx=idx)
    lanes = []
    for k, a in enumerate(ALPHAS):
        meta = json.load(open(os.path.join(WORK, "s28", f"lane{k}.json")))
        r = np.fromfile(os.path.join(WORK, "s28", f"ranks{k}.f64"), dtype=np.float64)
        assert r.size == N
        top = np.argsort(-r, kind="stable")[:4096]
        blocks = r.reshape(-1, BLOCK)
        arrays[f"lane{k}_sample"] = r[idx]
        arrays[f"lane{k}_top_idx"] = top.astype(np.int64)
        arrays[f"lane{k}_top"] = r[top]
        arrays[f"lane{k}_block_sum"] = np.sum(blocks.astype(np.longdouble), axis=1).astype(np.float64)
        arrays[f"lane{k}_block_max"] = blocks.max(axis=1)
        arrays[f"lane{k}_trace"] = np.asarray(meta["err_trace"], np.float64)
        lanes.append(dict(alpha=a, iterations=meta["iterations"], converged=meta["converged"],
                          loop_ms=meta["loop_ms"], total=float(np.sum(r.astype(np.longdouble))),
                          projections=projections(r)))
        print(f"alpha {a}: {meta['iterations']} iterations, converged {meta['converged']}", flush=True)
        del r, blocks
    np.savez_compressed(os.path.join(GOLD, "c5_rmat28.npz"), **arrays)
    with open(os.path.join(GOLD, "c5_rmat28.json"), "w") as f:
        json.dump(dict(config="rmat28 alphas .95/.85/.75 tau 1e-6 L2 max 500 (reference pagerank, "
                              "pagerank.hpp:70-108; graph by oracle/csr_inplace.hpp, fingerprint-pinned "
                              "to build_csr at scales 22 and 26)",
                       seed=2108, graph=fp, lanes=lanes, block=BLOCK), f, indent=1)
    print("c5 written")


if __name__ == "__main__":
    {"run": run, "summarize": summarize}[sys.argv[1] if len(sys.argv) > 1 else "summarize"]()
