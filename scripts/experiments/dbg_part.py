import numpy as np, ctypes as C
import paper_2108_02997_b200 as prl
from paper_2108_02997_b200 import distributed, _lib
from paper_2108_02997_b200._lib import lib, check
import torch
g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
al=[0.5,0.85]
want = prl.pagerank_batched(g, al, 1e-9)
print("fused trace", want.trace[:5, :, 0])
for nr in [1, 2]:
    parts = [distributed._Part(g, al, 1e-9, prl.NormKind.L1, 500, 0, r, nr, 0) for r in range(nr)]
    for p in parts: p.set_stream(); p.init()
    for it in range(5):
        pars = [p.step() for p in parts]; par = pars[0]
        torch.cuda.synchronize()
        sl = [p.slot.clone() for p in parts]
        for dst in parts:
            for r, src in enumerate(parts):
                if src is not dst:
                    dst.chunk(par, r).copy_(src.chunk(par, r)); dst.slot[r].copy_(src.slot[r])
        for p in parts: p.finalize()
        torch.cuda.synchronize()
        if it < 2: print("nr", nr, "it", it, "rank partial rows L1/dang:", [s[:, :].cpu().numpy().round(6).tolist() for s in sl][0])
    K=2; trace=np.zeros((500,K,4)); its=np.zeros(K,np.int32)
    r=_lib.Result(None, its.ctypes.data_as(C.POINTER(C.c_int)), None, None, trace.ctypes.data_as(C.POINTER(C.c_double)), 0.0, 0)
    check(lib().prgpu_session_results(parts[0]._s, C.byref(r)))
    print("nr", nr, "trace", trace[:5, :, 0])
