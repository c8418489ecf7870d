"""Graph-loop step time of a bench config (the bench's `value` path) for A/B
runs of different builds (PRGPU_LIB=...) or switches: median of N steps."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import paper_2108_02997_b200 as prl  # noqa
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
if cfg["kind"] == "rmat":
    g = prl.generate_rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, bench.SEED)
else:
    g = prl.generate_grid(cfg["side"], 0.6, 0.01, bench.SEED)
s = prl.Session(g, cfg["alphas"], cfg["tol"], prl.NormKind(cfg["norm"]), 500, cfg.get("stop_mask", 0))
for _ in range(2):
    s.run()
ms = [s.run() for _ in range(steps)]
print(f"{os.environ.get('PRGPU_LIB', 'current')}: step median {statistics.median(ms):.2f} ms  min {min(ms):.2f}  "
      f"all {[round(x, 1) for x in ms]}")
