"""A/B of the segmented hub pull on a bench config: the graph is built once,
then one session per variant (a space-separated list of VAR=value settings
read at session creation; "" = the defaults).  Per variant: the graph-loop
step time (median of N), the in-graph kernel time of every iteration, and the
run compared with the first variant's (iterations, ranks on a sample).
  python scripts/seg_ab.py c5 6 "PRGPU_SEG=0" "PRGPU_SEG=1" "PRGPU_SEG=1 PRGPU_SEG_T=256"
"""
import os, sys, statistics, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import paper_2108_02997_b200 as prl  # noqa

cfg = bench.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2])
variants = sys.argv[3:] or [""]
t0 = time.time()
if cfg["kind"] == "rmat":
    g = prl.generate_rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, bench.SEED)
else:
    g = prl.generate_grid(cfg["side"], 0.6, 0.01, bench.SEED)
print(f"graph: N={g.vertex_count} E={g.edge_count()} built in {time.time() - t0:.1f} s", flush=True)
base = None
rs = np.random.default_rng(5)
sample = rs.integers(0, g.vertex_count, 1 << 16)
for v in variants:
    sets = dict(kv.split("=", 1) for kv in v.split())
    old = {k: os.environ.get(k) for k in sets}
    os.environ.update(sets)
    try:
        t0 = time.time()
        s = prl.Session(g, cfg["alphas"], cfg["tol"], prl.NormKind(cfg["norm"]), 500, cfg.get("stop_mask", 0))
        t_create = time.time() - t0
        for _ in range(2):
            s.run()
        ms = [s.run() for _ in range(steps)]
        kt = s.kernel_times()
        want = cfg["scale"] <= 26 if cfg["kind"] == "rmat" else True
        res = s.results(want_ranks=want)
        its = res["iterations"].tolist()
        line = (f"[{v or 'defaults'}] step median {statistics.median(ms):.2f} ms min {min(ms):.2f}; "
                f"create {t_create:.2f} s; iterations {its}; kernel ms/iter {np.round(kt, 2).tolist()}")
        cur = dict(its=its, trace=res["trace"].copy(),
                   ranks=res["ranks"][:, sample].copy() if want else None)
        if base is None:
            base = cur
        else:
            tr = float(np.nanmax(np.abs(cur["trace"][: len(base["trace"])] / base["trace"] - 1.0))) \
                if cur["trace"].shape == base["trace"].shape else float("nan")
            line += f"; vs first: iterations {'==' if cur['its'] == base['its'] else '!='}, trace rel {tr:.2e}"
            if want:
                line += f", ranks Linf {float(np.max(np.abs(cur['ranks'] - base['ranks']))):.2e}"
        print(line, flush=True)
        s.close()
    finally:
        for k, o in old.items():
            if o is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = o
