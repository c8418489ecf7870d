#!/usr/bin/env python3
"""Turn gpurun_out/ evidence (scripts/gpu_bench_r1.sh) into tracked profiles/.

    python scripts/collect_profiles.py r1
writes profiles/<tag>_bench.json, <tag>_launches.md, <tag>_ncu_pull.json and
profiles/traffic.json (DRAM bytes per pull launch, read by bench.py).
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summary  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(fn):
    rows = list(csv.reader(open(fn)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / 1e6:.3f} | {100 * sum(v) / tot:.1f}% | "
                     f"{sum(v) / len(v) / 1e3:.1f} |")
    return tot, lines


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    bench = [l for l in open(os.path.join(OUT, "bench_full.log")) if l.startswith("{")][-1]
    with open(os.path.join(PROF, f"{tag}_bench.json"), "w") as f:
        f.write(bench)
    md = [f"# {tag}: ncu launch lists (`gpu__time_duration.sum`, `--clock-control none`)", "",
          "Cold-cache, serialised per-launch times: compare shares, not absolutes.", ""]
    for fn, title in [("launches_c2.csv", "bench.py --steps 1 --warmup 3 (PRGPU_NO_GRAPH=1: "
                       "host-driven launches so ncu sees each pull launch)"),
                      ("graphs_c2.csv", "same command with the CUDA graph, `--graph-profiling graph` "
                       "(one entry per WHILE-loop graph = one sweep)")]:
        p = os.path.join(OUT, fn)
        if os.path.exists(p):
            tot, lines = launches(p)
            md += [f"## {title}", "", f"total {tot / 1e6:.3f} ms", ""] + lines + [""]
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(md))
    rep = os.path.join(OUT, f"{tag}_c2_pull.ncu-rep")
    kernels = summary(rep)  # the kernels of one all-lanes-live iteration (hub chunks, packed + empty)
    with open(os.path.join(PROF, f"{tag}_ncu_pull.json"), "w") as f:
        json.dump(kernels if len(kernels) > 1 else kernels[0], f, indent=1)

    def to_bytes(s, k):
        v, u = s[k].split()[:2]
        return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    traffic = sum(to_bytes(s, "dram__bytes_read.sum") + to_bytes(s, "dram__bytes_write.sum") for s in kernels)
    tp = os.path.join(PROF, "traffic.json")
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old["c2"] = traffic  # the other configs' entries (ncu captures of their own) are kept
    old["source"] = (f"profiles/{tag}_ncu_pull.json (ncu --set full of the pull kernels of one C2 "
                     "iteration, all 11 lanes active; summed)")
    with open(tp, "w") as f:
        json.dump(old, f, indent=1)
    print("profiles written; pull traffic per launch", traffic / 1e9, "GB")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
