"""Time the pieces of the e2e path (C ABI with host buffers) on the C2 graph."""
import ctypes as C, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2108_02997_b200 as prl
from paper_2108_02997_b200 import _lib
L = _lib.lib()
g = prl.generate_rmat(22, 16, 0.57, 0.19, 0.19, 2108)
n, e = g.vertex_count, g.edge_count()
off = torch.from_numpy(g.in_offsets).pin_memory(); nbr = torch.from_numpy(g.in_neighbors).pin_memory()
deg = torch.from_numpy(g.out_degree).pin_memory()
alphas = [0.5 + 0.05 * i for i in range(11)]
K = 11
ranks = torch.empty((K, n), dtype=torch.float64).pin_memory()
its = np.zeros(K, np.int32)
a = (C.c_double * K)(*alphas)
p = _lib.Params(K, a, None, 1e-6, 0, 0, 500, None)
for rep in range(3):
    t0 = time.perf_counter()
    h = C.c_void_p(); _lib.check(L.prgpu_graph_from_csr(n, off.data_ptr(), nbr.data_ptr(), deg.data_ptr(), 0, C.byref(h)))
    t1 = time.perf_counter()
    s = C.c_void_p(); _lib.check(L.prgpu_session_create(h, C.byref(p), C.byref(s)))
    t2 = time.perf_counter()
    ms = C.c_double(); _lib.check(L.prgpu_session_run(s, C.byref(ms)))
    t3 = time.perf_counter()
    r = _lib.Result(C.cast(ranks.data_ptr(), C.POINTER(C.c_double)), its.ctypes.data_as(C.POINTER(C.c_int)), None, None, None, 0.0, 0)
    _lib.check(L.prgpu_session_results(s, C.byref(r)))
    t4 = time.perf_counter()
    L.prgpu_session_free(s); L.prgpu_graph_free(h)
    t5 = time.perf_counter()
    print(f"from_csr {1e3*(t1-t0):.1f} ms  session {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f} (loop {ms.value:.1f})  results {1e3*(t4-t3):.1f}  free {1e3*(t5-t4):.1f}")
