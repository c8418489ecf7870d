"""Box probe: host cores/RAM, and the reference pagerank's per-iteration time on
the C5 graph (generated on the GPU, downloaded in the reference layout)."""
import os, sys, time, threading, json, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
print(subprocess.run("nproc; free -g; lscpu | grep -i 'model name\\|^CPU(s)\\|NUMA\\|Thread'; nvidia-smi --query-gpu=name,memory.total --format=csv", shell=True, capture_output=True, text=True).stdout, flush=True)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
import paper_2108_02997_b200 as prl
from pyoracle import Ref
t = time.time(); g = prl.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 2108); print("gen", time.time() - t, flush=True)
t = time.time(); off, nbr, deg = g.in_offsets, g.in_neighbors, g.out_degree; print("download", time.time() - t, flush=True)
n = g.vertex_count; del g
R = Ref()
t = time.time(); h = R.csr_from_arrays(n, off, nbr, deg); print("ref csr", time.time() - t, flush=True)
e = int(off[-1]); del nbr
for lanes in (1, 3):
    out = [None] * lanes
    def work(i):
        out[i] = R.pagerank(h, [0.95, 0.85, 0.75][i], 1e-300, "l2", 1, want_ranks=False)
    ts = [threading.Thread(target=work, args=(i,)) for i in range(lanes)]
    t0 = time.perf_counter()
    [x.start() for x in ts]; [x.join() for x in ts]
    dt = time.perf_counter() - t0
    print(json.dumps(dict(lanes=lanes, wall_s=dt, loop_ms=[o["elapsed_ms"] for o in out], gteps=lanes * e / dt / 1e9)), flush=True)
