"""Sharded graph build (SURVEY 8e set-up; prgpu_graph_generate_rmat_shard):
every rank generates all edges slab by slab, computes the exact global
degrees (so its relabelled vertex arrays equal the whole graph's) and keeps
only the in-edges of its contiguous engine-row range.  Checked against the
whole-graph build and the single-GPU run: shards tile the rows and edges,
vertex arrays are identical, and an N-rank partitioned run over the shards
(emulated on one GPU, fused peer exchange and the buffer-copy exchange)
gives the single-GPU iterations and ranks (1e-13)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHAS = [0.95, 0.85, 0.6]


def perm(prl, g):
    p = np.zeros(g.vertex_count, np.uint32)
    prl._lib.check(prl._lib.lib().prgpu_graph_permutation(g.handle, p.ctypes.data), "perm")
    return p


@pytest.mark.parametrize("scale,nranks,slab", [(16, 2, 1 << 17), (18, 3, 1 << 20), (18, 2, 0)])
def test_shards_tile_the_graph_and_match_single_gpu(prl, monkeypatch, scale, nranks, slab):
    from paper_2108_02997_b200 import distributed
    if slab:  # several slabs per pass (the C5 build uses 4)
        monkeypatch.setenv("PRGPU_SLAB_KEYS", str(slab))
    full = prl.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 2108)
    shards = [prl.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 2108, shard=(r, nranks)) for r in range(nranks)]
    info = [s.shard_info() for s in shards]
    assert info[0]["row_begin"] == 0 and info[-1]["row_end"] == full.vertex_count
    for a, b in zip(info, info[1:]):
        assert a["row_end"] == b["row_begin"]
    assert sum(i["local_edges"] for i in info) == full.edge_count()
    assert max(i["local_edges"] for i in info) < 0.75 * full.edge_count()
    p = perm(prl, full)
    for s in shards:
        assert s.edge_count() == full.edge_count() and s.vertex_count == full.vertex_count
        assert int(s.info.dangling_count) == int(full.info.dangling_count)
        assert np.array_equal(perm(prl, s), p)
        assert np.array_equal(s.out_degree_only(), full.out_degree_only())
    with pytest.raises(ValueError):  # a shard cannot run alone
        prl.pagerank(shards[0], prl.PageRankConfig())
    single = prl.pagerank_batched(full, ALPHAS, 1e-9, prl.NormKind.L2, 300)
    sent = {}
    for fused, need in ((True, "1"), (True, "0"), (False, "1")):
        monkeypatch.setenv("PRGPU_NEED", need)  # 0: every row to every peer
        res = distributed.emulate(shards[0], ALPHAS, nranks, 1e-9, prl.NormKind.L2, 300, want_ranks=True,
                                  fused=fused, shards=shards)
        sent[(fused, need)] = res.sent_bytes
        for k, r in enumerate(single.results):
            assert int(res.iterations[k]) == r.iterations, (fused, k)
            assert float(np.max(np.abs(res.ranks[k] - r.ranks))) <= 1e-13, (fused, k)
    # the OR-reduced needed-only mask (prgpu_part_need_local / set_need) sends fewer rows
    assert 0 < sent[(True, "1")] < sent[(True, "0")]


def device_bytes(prl, g=None, sess=None):
    import ctypes as C
    gb, sb = C.c_uint64(), C.c_uint64()
    prl._lib.check(prl._lib.lib().prgpu_device_bytes(g.handle if g else None, sess, C.byref(gb), C.byref(sb)),
                   "device bytes")
    return gb.value, sb.value


@pytest.mark.slow
def test_c5_shards_cut_the_per_rank_edges_and_ranks(prl):
    """C5 (RMAT-28, K = 3) at 2 ranks, per rank (prgpu_device_bytes): the
    shard holds about half the in-edges and the partition session only its
    rows' ranks, against the same session on the whole graph; the vertex
    arrays (and the contribution replica every rank gathers from, caller
    memory) stay whole, as SURVEY 8e's set-up has them."""
    from paper_2108_02997_b200 import distributed
    full = prl.generate_rmat(28, 16, 0.57, 0.19, 0.19, 2108)
    e = full.edge_count()
    pfull = perm(prl, full)
    pf = distributed._Part(full, ALPHAS, 1e-6, prl.NormKind.L2, 500, 0, 0, 2, 0)
    g_full, s_full = device_bytes(prl, full, pf._s)
    pf.close()
    del pf, full
    per_rank, local = [], []
    for r in range(2):
        sh = prl.generate_rmat(28, 16, 0.57, 0.19, 0.19, 2108, shard=(r, 2))
        info = sh.shard_info()
        assert sh.edge_count() == e
        assert np.array_equal(perm(prl, sh), pfull)
        ps = distributed._Part(sh, ALPHAS, 1e-6, prl.NormKind.L2, 500, 0, r, 2, 0)
        per_rank.append(device_bytes(prl, sh, ps._s))
        local.append(info["local_edges"])
        ps.close()
        del ps, sh
    assert sum(local) == e and max(local) < 0.6 * e
    col_full = 4 * e
    for (g_sh, s_sh), le in zip(per_rank, local):
        assert g_full - g_sh >= 0.9 * 4 * (e - le), (g_full, g_sh)  # only the shard's edges held
        assert s_sh < s_full
    worst = max(g + s for g, s in per_rank)
    assert worst <= 0.8 * (g_full + s_full), (worst, g_full + s_full)
    print(f"C5 at N=2, per rank: whole graph {g_full / 1e9:.1f} GB + session {s_full / 1e9:.1f} GB; shards "
          + ", ".join(f"{g / 1e9:.1f} + {s / 1e9:.1f} GB" for g, s in per_rank)
          + f" (in-edges {col_full / 1e9:.1f} -> " + ", ".join(f"{4 * x / 1e9:.1f}" for x in local) + " GB)")
