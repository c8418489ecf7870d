"""Time the pieces of the e2e path (C ABI, pinned host buffers) on a bench
config's graph: python scripts/e2e_probe.py c5 [reps]  (PRGPU_TIMING_LOG=1
adds the library's phase marks on stderr)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2108_02997_b200 as prl  # noqa: E402
from paper_2108_02997_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = _lib.lib()
g = prl.generate_rmat(cfg["scale"], 16, 0.57, 0.19, 0.19, bench.SEED)
n, e = g.vertex_count, g.edge_count()
off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
nbr = torch.empty(e, dtype=torch.int32, pin_memory=True)
deg = torch.empty(n, dtype=torch.int32, pin_memory=True)
_lib.check(L.prgpu_graph_download(g.handle, off.data_ptr(), nbr.data_ptr(), deg.data_ptr(), None))
del g
K = len(cfg["alphas"])
ranks = torch.empty((K, n), dtype=torch.float64, pin_memory=True)
its = np.zeros(K, np.int32)
a = (C.c_double * K)(*cfg["alphas"])
p = _lib.Params(K, a, None, cfg["tol"], cfg["norm"], cfg.get("stop_mask", 0), 500, None)
for rep in range(reps):
    t0 = time.perf_counter()
    h = C.c_void_p()
    _lib.check(L.prgpu_graph_from_csr(n, off.data_ptr(), nbr.data_ptr(), deg.data_ptr(), 0, C.byref(h)))
    t1 = time.perf_counter()
    s = C.c_void_p()
    _lib.check(L.prgpu_session_create(h, C.byref(p), C.byref(s)))
    t2 = time.perf_counter()
    ms = C.c_double()
    _lib.check(L.prgpu_session_run(s, C.byref(ms)))
    t3 = time.perf_counter()
    r = _lib.Result(C.cast(ranks.data_ptr(), C.POINTER(C.c_double)), its.ctypes.data_as(C.POINTER(C.c_int)),
                    None, None, None, 0.0, 0)
    _lib.check(L.prgpu_session_results(s, C.byref(r)))
    t4 = time.perf_counter()
    L.prgpu_session_free(s)
    L.prgpu_graph_free(h)
    t5 = time.perf_counter()
    rr = _lib.Result(C.cast(ranks.data_ptr(), C.POINTER(C.c_double)), its.ctypes.data_as(C.POINTER(C.c_int)),
                     None, None, None, 0.0, 0)
    h = C.c_void_p()
    t6 = time.perf_counter()
    _lib.check(L.prgpu_graph_from_csr(n, off.data_ptr(), nbr.data_ptr(), deg.data_ptr(), 0, C.byref(h)))
    _lib.check(L.prgpu_pagerank(h, C.byref(p), C.byref(rr)))
    L.prgpu_graph_free(h)
    t7 = time.perf_counter()
    print(f"from_csr {1e3*(t1-t0):.1f} ms  session {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f} "
          f"(loop {ms.value:.1f})  results {1e3*(t4-t3):.1f}  free {1e3*(t5-t4):.1f} | e2e one call "
          f"{1e3*(t7-t6):.1f} ms", flush=True)
