import os, numpy as np
import paper_2108_02997_b200 as prl
g1 = prl.generate_rmat(20, 16, 0.57, 0.19, 0.19, 2108)
os.environ["PRGPU_ROW_SORT"] = "0"
g2 = prl.csr_from_arrays(g1.vertex_count, g1.in_offsets, g1.in_neighbors, g1.out_degree)
a = prl.pagerank_batched(g1, [0.85], 1e-9, prl.NormKind.L1, 200)
b = prl.pagerank_batched(g2, [0.85], 1e-9, prl.NormKind.L1, 200)
print("unsorted differs:", not np.array_equal(a.results[0].ranks, b.results[0].ranks), np.max(np.abs(a.results[0].ranks-b.results[0].ranks)))
