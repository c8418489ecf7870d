"""The segmented hub pull (SegPlan: the in-edges of the high in-degree rows
regrouped into (row, source segment) pieces pulled segment by segment, each
piece's partial combined in segment order by the row's epilogue) against the
oracle and against the unsegmented pull.  Small graphs never pick it by
themselves (their contribution table fits L2), so the tests force it with tiny
segments: every path runs — wide pieces cut into chunks with the hand-off,
small-piece runs, combine tasks, the cold rest segment, every lane-width mode.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RANK_TOL = 1e-10


def nk(prl, name):
    return {"l1": prl.NormKind.L1, "l2": prl.NormKind.L2, "linf": prl.NormKind.LInf}[name]


def edge_list(prl, n, pairs):
    return prl.EdgeList(n, np.asarray(pairs, np.uint32).reshape(-1, 2))


SEG_ENVS = [
    # segment KB, hot segments, least in-degree, chunk edges
    dict(PRGPU_SEG_KB="16", PRGPU_SEG_HOT="3", PRGPU_SEG_T="300"),    # cold rest, mostly small pieces
    dict(PRGPU_SEG_KB="256", PRGPU_SEG_HOT="63", PRGPU_SEG_T="600", PRGPU_CHUNK="512",
         PRGPU_SEG_PMIN="0"),                                         # every segment hot, chunked wide pieces, no folding
    dict(PRGPU_SEG_KB="4", PRGPU_SEG_HOT="40", PRGPU_SEG_T="257", PRGPU_SEG_PMIN="20"),  # tiny segments, most pieces folded
    dict(PRGPU_SEG_KB="32", PRGPU_SEG_HOT="8", PRGPU_SEG_T="24"),     # packed rows segmented too
]


@pytest.mark.parametrize("env", SEG_ENVS)
def test_segmented_pull_matches_oracle_and_plain(prl, oracle, monkeypatch, env):
    n, pairs = oracle.rmat(17, 16, 0.57, 0.19, 0.19, 2108)
    h = oracle.build_csr_handle(n, pairs)
    g = prl.build_csr(edge_list(prl, n, pairs))
    eleven = [0.5 + 0.05 * i for i in range(11)]
    try:
        monkeypatch.setenv("PRGPU_SEG", "0")
        one3 = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        one11 = prl.pagerank_batched(g, eleven, 1e-6, prl.NormKind.L1, 300)
        monkeypatch.setenv("PRGPU_SEG", "1")
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        for norm in ("l1", "l2", "linf"):
            want = oracle.pagerank(h, 0.85, 1e-9, norm, 300)
            got = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-9, nk(prl, norm), 300))
            assert got.iterations == want["iterations"], norm
            assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, norm
            assert abs(got.ranks.sum() - 1.0) <= 1e-9
        two3 = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        for a, b, alpha in zip(one3.results, two3.results, (0.95, 0.85, 0.6)):
            assert a.iterations == b.iterations
            assert np.max(np.abs(a.ranks - b.ranks)) <= 1e-15
            want = oracle.pagerank(h, alpha, 1e-9, "l2", 300)
            assert b.iterations == want["iterations"]
            assert np.max(np.abs(b.ranks - want["ranks"])) <= RANK_TOL
        two11 = prl.pagerank_batched(g, eleven, 1e-6, prl.NormKind.L1, 300)
        for a, b in zip(one11.results, two11.results):
            assert a.iterations == b.iterations and np.max(np.abs(a.ranks - b.ranks)) <= 1e-15
        # bit-reproducible (sweep.hpp:176-179): a second segmented run, and the
        # host-driven launches instead of the CUDA graph
        again = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        monkeypatch.setenv("PRGPU_NO_GRAPH", "1")
        hosted = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        for a, b, c in zip(two3.results, again.results, hosted.results):
            assert a.iterations == b.iterations == c.iterations
            assert np.array_equal(a.ranks, b.ranks) and np.array_equal(a.ranks, c.ranks)
    finally:
        oracle.free_csr(h)


def test_segmented_pull_series_and_observer(prl, oracle, monkeypatch):
    """The other entry points over a segmented session: the power-series
    sweep (a K = 1 chain) and the observed run."""
    n, pairs = oracle.rmat(16, 16, 0.57, 0.19, 0.19, 7)
    h = oracle.build_csr_handle(n, pairs)
    g = prl.build_csr(edge_list(prl, n, pairs))
    try:
        monkeypatch.setenv("PRGPU_SEG", "1")
        monkeypatch.setenv("PRGPU_SEG_KB", "8")
        monkeypatch.setenv("PRGPU_SEG_HOT", "5")
        monkeypatch.setenv("PRGPU_SEG_T", "300")
        alphas = [0.9, 0.85, 0.5]
        ser = prl.pagerank_batched(g, alphas, 1e-8, prl.NormKind.L1, 300, series=True)
        for r, alpha in zip(ser.results, alphas):
            want = oracle.pagerank(h, alpha, 1e-8, "l1", 300)
            assert r.iterations == want["iterations"]
            assert np.max(np.abs(r.ranks - want["ranks"])) <= RANK_TOL
        seen = []
        got = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-8, prl.NormKind.LInf, 300),
                           lambda it, ranks, err: seen.append((it, err, float(ranks.sum()))))
        want = oracle.pagerank(h, 0.85, 1e-8, "linf", 300)
        assert got.iterations == want["iterations"] == len(seen)
        assert all(abs(s - 1.0) <= 1e-9 for _, _, s in seen)
        assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL
    finally:
        oracle.free_csr(h)


@pytest.mark.parametrize("K", [2, 5, 8, 16])
def test_segmented_pull_lane_counts_ref_trace_and_caps(prl, oracle, monkeypatch, K):
    """Every lane-count instance of the three segmented kernels, with the
    L1-vs-reference trace (sweep.hpp:193-196), all-norm stopping and an
    iteration cap, against the unsegmented run of the same session
    parameters."""
    n, pairs = oracle.rmat(15, 16, 0.57, 0.19, 0.19, 11)
    g = prl.build_csr(edge_list(prl, n, pairs))
    alphas = [0.5 + 0.5 * k / K for k in range(K)]
    ref = prl.reference_ranks(g)
    runs = {}
    for seg in ("0", "1"):
        monkeypatch.setenv("PRGPU_SEG", seg)
        monkeypatch.setenv("PRGPU_SEG_KB", "8")
        monkeypatch.setenv("PRGPU_SEG_HOT", "6")
        runs[seg] = (
            prl.pagerank_batched(g, alphas, 1e-9, prl.NormKind.LInf, 300, stop_mask=7, ref_ranks=ref),
            prl.pagerank_batched(g, alphas, 1e-12, prl.NormKind.L2, 7),  # capped: nothing converges
        )
    for a, b in zip(runs["0"], runs["1"]):
        assert a.run_iterations == b.run_iterations
        for x, y in zip(a.results, b.results):
            assert x.iterations == y.iterations and x.converged == y.converged
            assert np.max(np.abs(x.ranks - y.ranks)) <= 1e-15
        ta, tb = a.trace[: a.run_iterations], b.trace[: b.run_iterations]
        live = ~np.isnan(ta)
        assert np.array_equal(live, ~np.isnan(tb))
        # (norms of 1e-12 carry the summation order's rounding, ~1e-18 absolute)
        assert np.all(np.abs(ta[live] - tb[live]) <= 1e-9 * np.abs(ta[live]) + 1e-16)
    assert not any(r.converged for r in runs["1"][1].results)
