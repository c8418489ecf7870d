#!/usr/bin/env python3
"""gpurun_out/r2/ (scripts/gpu_refresh.sh) -> profiles/r2_*: every config's
bench line (r2_configs.{json,md}, r2_bench_c5.json, r2_bench_reference_c5.json),
the C5 launch list (r2_launches_c5.{csv,md}), the ncu --set full summary of
one C5 iteration's kernels (r2_ncu_c5_seg.json) and profiles/traffic.json."""
import csv, glob, json, os, shutil, sys
from collections import defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summary  # noqa: E402
SRC, PROF = os.path.join(ROOT, "gpurun_out", "r2"), os.path.join(ROOT, "profiles")


def last_json(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


lines = {}
for f in sorted(glob.glob(os.path.join(SRC, "bench_*.log")) + glob.glob(os.path.join(SRC, "ref_*.log"))):
    d = last_json(f)
    if d:
        lines[os.path.basename(f)[:-4]] = d
json.dump(lines, open(os.path.join(PROF, "r2_configs.json"), "w"), indent=1)
if "bench_c5" in lines:
    json.dump(lines["bench_c5"], open(os.path.join(PROF, "r2_bench_c5.json"), "w"))
if "ref_c5" in lines and lines["ref_c5"]["cpu_baseline"]["cores"] >= 16:  # a full round of 16 concurrent lanes
    json.dump(lines["ref_c5"], open(os.path.join(PROF, "r2_bench_reference_c5.json"), "w"))
peak = lines.get("bench_c5", {}).get("roofline", {}).get("peak")
md = ["# r2: bench lines for every config at HEAD (one fresh B200, `scripts/gpu_refresh.sh`)", "",
      "`python bench.py --config <c> --steps 10 --warmup 3`; C5 (the default) is also `profiles/r2_bench_c5.json`.",
      "Raw JSON lines: `profiles/r2_configs.json`.  GTEPS = lane-iterations x E / step; frac = algorithmic",
      f"bytes per iteration / in-graph kernel time / {peak} GB/s; cpu = `cpu_baseline` (C1-C3 the reference itself,",
      "C4/C5 the bit-identical threaded port on 16 cores).", "",
      "| config | GTEPS | ms / step | roofline frac | e2e GTEPS (ms, p90) | cpu GTEPS (kind) | SM MHz, reasons |",
      "|---|---|---|---|---|---|---|"]
for k in ("c1", "c2", "c2k1", "c3", "c4", "c5", "c2series", "c5series"):
    d = lines.get("bench_" + k)
    if not d:
        continue
    r, e, c = d.get("roofline") or {}, d.get("e2e") or {}, d.get("cpu_baseline") or {}
    frac = f"{r['frac']:.3f}" if r.get("frac") else "-"
    e2e = f"{e['value']:.1f} ({e['ms_per_step']:.1f}, {e.get('ms_p90', 0):.1f})" if e.get("value") else "-"
    cpu = f"{c['value']:.3f} ({c.get('kind')})" if c.get("value") else "-"
    md.append(f"| {k} | {d['value']:.1f} | {d['ms_per_step']:.2f} | {frac} | {e2e} | {cpu} | "
              f"{d['clocks']['sm_mhz']}, {d['clocks']['reasons']} |")
refs = []
if "ref_c5" not in lines or lines["ref_c5"]["cpu_baseline"]["cores"] < 16:  # the committed 16-lane run
    lines["ref_c5"] = json.load(open(os.path.join(PROF, "r2_bench_reference_c5.json")))
for k in ("ref_c2", "ref_c5"):
    if k in lines:
        refs.append(f"{k[4:].upper()} {lines[k]['value']:.3f} GTEPS on {lines[k]['cpu_baseline']['cores']} host threads")
md += ["", "Reference arm (`--impl reference`): " + "; ".join(refs) + ".",
       "Series lines (`c2series`, `c5series`) count the separate runs' lane-iterations x E per second (`value_kind`); "
       "they run 22 / 13 K = 1 pulls instead of 173 / 33 lane-iterations."]
open(os.path.join(PROF, "r2_configs.md"), "w").write("\n".join(md) + "\n")

lc = os.path.join(SRC, "launches_c5.csv")
if os.path.exists(lc):
    shutil.copy(lc, os.path.join(PROF, "r2_launches_c5.csv"))
    rows = list(csv.reader(l for l in open(lc) if l.startswith('"')))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["# r2: C5 launch list (ncu `--metrics gpu__time_duration.sum --clock-control none`)", "",
           "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 "
           "--warmup 3 --no-e2e --no-cpu-baseline`",
           "(raw: `profiles/r2_launches_c5.csv`).  The bench's CUDA-graph loop runs its kernels inside conditional",
           "nodes, which ncu does not list; the pull kernels below are the bench's `time_pull` pass (host-driven,",
           "the kernels of the armed lane mode only) plus the graph and segment-plan builds.  Cold-cache and",
           "serialised per launch: compare shares, not absolute times.  pull_kernel PATHS (last template",
           "argument): 5 wide-piece chunks, 8 small-piece runs, 18 combine + packed + empty rows + finalize.", "",
           "| kernel | launches | total ms | ms / launch | share of listed |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:32]:
        out.append(f"| `{k[:78]}` | {len(v)} | {sum(v) / 1e6:.1f} | {sum(v) / len(v) / 1e6:.2f} | {100 * sum(v) / tot:.1f} % |")
    pull = sum(sum(v) for k, v in agg.items() if "pull_kernel" in k)
    out += ["", f"pull kernels: {pull / 1e6:.1f} ms of {tot / 1e6:.1f} ms listed ({100 * pull / tot:.1f} %)."]
    open(os.path.join(PROF, "r2_launches_c5.md"), "w").write("\n".join(out) + "\n")

rep = os.path.join(SRC, "c5_seg_full.ncu-rep")
if os.path.exists(rep):
    ks = summary(rep)
    json.dump(ks, open(os.path.join(PROF, "r2_ncu_c5_seg.json"), "w"), indent=1)

    def gb(x):
        v, u = x.split()[:2]
        return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]
    tr = sum(gb(k["dram__bytes_read.sum"]) + gb(k["dram__bytes_write.sum"]) for k in ks)
    tp = os.path.join(PROF, "traffic.json")
    t = json.load(open(tp))
    t["c5"] = tr
    t["source"] = ("DRAM read+write per all-lanes iteration from ncu --set full of the iteration's pull kernels "
                   "(c2: profiles/r1_ncu_pull.json; c5: profiles/r2_ncu_c5_seg.json, the three kernels of the "
                   "segmented pull, algorithmic bytes of that iteration 37.9 GB; 249.2 GB before the segmented pull: "
                   "profiles/r2_ncu_c5_hub.json + r2_ncu_c5_packed.json)")
    json.dump(t, open(tp, "w"), indent=1)
    print("c5 traffic per iteration: %.1f GB" % (tr / 1e9))
print("ok")
