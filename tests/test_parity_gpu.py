"""GPU parity: the CUDA path (through the C ABI) against the reference's goldens
and the oracle restatement on the same seeded inputs.

Bars (BASELINE.json north_star): CSR arrays bit-identical to build_csr;
iteration counts exactly equal (or +-1 only where the reference's final delta
is within 1e-3*tau of tau); ranks within Linf 1e-10 of the reference's.
"""
import math
import os

import numpy as np
import pytest

from conftest import GOLD, load_golden

pytestmark = pytest.mark.gpu

RANK_TOL = 1e-10  # Linf, fp64 (north_star)
NORMS = ["l1", "l2", "linf"]


def nk(prl, name):
    return {"l1": prl.NormKind.L1, "l2": prl.NormKind.L2, "linf": prl.NormKind.LInf}[name]


def iterations_match(got, want, trace, tol):
    """Exact, or +-1 where the reference's err at the crossing is within 1e-3*tau of tau."""
    if got == want:
        return True
    if abs(got - want) != 1:
        return False
    t = min(got, want)
    cand = [trace[i] for i in (t - 1, t) if 0 <= i < len(trace)]
    return any(abs(e - tol) <= 1e-3 * tol for e in cand)


def edge_list(prl, n, pairs):
    return prl.EdgeList(n, np.asarray(pairs, np.uint32).reshape(-1, 2))


# ---------------------------------------------------------------------------
def test_fixtures_csr_and_runs(prl, small_golden):
    for name, fx in small_golden["fixtures"].items():
        g = prl.build_csr(edge_list(prl, fx["n"], fx["pairs"]))
        assert g.in_offsets.tolist() == fx["csr"]["in_offsets"], name
        assert g.in_neighbors.tolist() == fx["csr"]["in_neighbors"], name
        assert g.out_degree.tolist() == fx["csr"]["out_degree"], name
        assert g.dangling.tolist() == fx["csr"]["dangling"], name
        for run in fx["runs"]:
            cfg = prl.PageRankConfig(run["alpha"], run["tol"], nk(prl, run["norm"]), run["max_iter"])
            r = prl.pagerank(g, cfg)
            assert iterations_match(r.iterations, run["iterations"], run["err_trace"], run["tol"]), \
                (name, run["alpha"], run["norm"], r.iterations, run["iterations"])
            assert r.converged == run["converged"]
            assert np.max(np.abs(r.ranks - np.array(run["ranks"]))) <= RANK_TOL


def test_acceptance_trials(prl, small_golden):
    """acceptance.cpp:104-132: 220 random digraphs (seed 4242, half with forced
    dangling vertices) against the reference's results and the dense oracle."""
    for i, t in enumerate(small_golden["trials"]):
        g = prl.build_csr(edge_list(prl, t["n"], t["pairs"]))
        cfg = prl.PageRankConfig(t["alpha"], t["tol"], nk(prl, t["norm"]), 500)
        r = prl.pagerank(g, cfg)
        assert iterations_match(r.iterations, t["iterations"], t["err_trace"], t["tol"]), i
        assert np.max(np.abs(r.ranks - np.array(t["ranks"]))) <= RANK_TOL, i
        assert np.max(np.abs(r.ranks - np.array(t["dense_ranks"]))) <= 1e-8, i


def test_known_answers(prl):
    el = lambda n, e: prl.EdgeList(n, np.array(e, np.uint32).reshape(-1, 2))  # noqa: E731
    two = prl.build_csr(el(2, [[0, 1], [1, 0]]))
    for a in (0.0, 0.5, 0.85, 1.0):  # test_pagerank.cpp:49-58
        r = prl.pagerank(two, prl.PageRankConfig(alpha=a))
        assert r.iterations == 1 and r.converged and np.allclose(r.ranks, 0.5, rtol=1e-12)
    one = prl.build_csr(prl.EdgeList(1))  # :60-67
    r = prl.pagerank(one, prl.PageRankConfig(alpha=0.85))
    assert r.iterations == 1 and r.converged and abs(r.ranks[0] - 1.0) <= 1e-14
    star = prl.build_csr(el(3, [[1, 0], [2, 0]]))  # :69-87
    r = prl.pagerank(star, prl.PageRankConfig(0.85, 1e-10))
    c = 1.0 / (3.0 + 2 * 0.85)
    assert r.converged and np.allclose(r.ranks, [(1 + 1.7) * c, c, c], rtol=1e-6)
    for bad in (dict(alpha=1.5), dict(alpha=-0.1), dict(tolerance=0.0), dict(max_iterations=0)):
        with pytest.raises(ValueError):  # :89-100
            prl.pagerank(two, prl.PageRankConfig(**bad))
    # graph.hpp:204-234: vertex_count 0 builds the empty graph; pagerank()
    # rejects it (pagerank.hpp:74) after validating the config (:73)
    empty = prl.build_csr(prl.EdgeList(0))
    assert empty.vertex_count == 0 and empty.edge_count() == 0
    assert empty.in_offsets.tolist() == [0] and empty.dangling.size == 0
    with pytest.raises(ValueError, match="no vertices"):
        prl.pagerank(empty, prl.PageRankConfig())
    with pytest.raises(ValueError, match="alpha"):
        prl.pagerank(empty, prl.PageRankConfig(alpha=2.0))
    # iteration cap honesty (:228-237)
    web = prl.build_csr(el(6, [[0, 1], [0, 2], [1, 2], [2, 0], [3, 2], [4, 0], [4, 3], [2, 4], [1, 5]]))
    r = prl.pagerank(web, prl.PageRankConfig(1.0, 1e-15, prl.NormKind.L1, 50))
    assert r.iterations == 50 and not r.converged
    r = prl.pagerank(web, prl.PageRankConfig(0.85, 1e-12, prl.NormKind.L1, 2))
    assert r.iterations == 2 and not r.converged
    # reference error (:239-261)
    assert prl.reference_error(star, prl.reference_ranks(star)) == 0.0
    e75 = prl.pagerank(star, prl.PageRankConfig(0.75, 1e-12))
    c75, c85 = 1 / (3 + 1.5), 1 / (3 + 1.7)
    expected = abs(2.5 * c75 - 2.7 * c85) + 2 * abs(c75 - c85)
    assert math.isclose(prl.reference_error(star, e75.ranks), expected, rel_tol=1e-4)


def test_ring_single_iteration(prl, oracle):
    """acceptance.cpp:248-259: k-regular ring, 1 iteration for every tau and norm."""
    n, pairs = oracle.regular_ring(100000, 3)
    g = prl.build_csr(edge_list(prl, n, pairs))
    assert g.dangling.size == 0
    for norm in prl.all_norms:
        for tol in prl.default_tolerance_grid():
            r = prl.pagerank(g, prl.PageRankConfig(0.85, tol, norm))
            assert r.iterations == 1 and r.converged


def test_observer_rank_conservation_and_floor(prl, oracle):
    """test_pagerank.cpp:118-146, acceptance.cpp:134-161: sum = 1 +- 1e-9 and the
    teleport floor on every iteration, seen through the observer."""
    rng = oracle.mt19937(11)
    for trial in range(8):
        n, pairs = oracle.random_digraph(rng, 2 + trial * 5, 0.2, True)
        g = prl.build_csr(edge_list(prl, n, pairs))
        seen = []

        def obs(it, ranks, err):
            seen.append(it)
            assert abs(float(np.sum(ranks.astype(np.longdouble))) - 1.0) <= 1e-9
            assert np.all(ranks >= (1 - 0.85) / n * (1 - 1e-12))

        r = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-9), obs)
        assert seen == list(range(1, r.iterations + 1))


def test_norm_and_alpha_ordering(prl, oracle):
    rng = oracle.mt19937(17)
    for trial in range(6):
        n, pairs = oracle.random_digraph(rng, 3 + 7 * trial, 0.2, True)
        g = prl.build_csr(edge_list(prl, n, pairs))
        for a in (0.7, 0.85, 0.95):
            its = [prl.pagerank(g, prl.PageRankConfig(a, 1e-6, nm)).iterations for nm in prl.all_norms]
            assert its[2] <= its[1] <= its[0]
        prev = 0
        for a in prl.default_damping_grid():
            it = prl.pagerank(g, prl.PageRankConfig(a, 1e-6)).iterations
            assert it >= prev
            prev = it


def test_error_norm_device(prl):
    r, s = [0.3, 0.7], [0.5, 0.5]
    assert math.isclose(prl.error_norm(prl.NormKind.L1, r, s), 0.4, rel_tol=1e-12)
    assert math.isclose(prl.error_norm(prl.NormKind.LInf, r, s), 0.2, rel_tol=1e-12)
    assert math.isclose(prl.error_norm(prl.NormKind.L2, r, s), math.sqrt(0.08), rel_tol=1e-12)
    with pytest.raises(ValueError):
        prl.error_norm(prl.NormKind.L1, [0.5, 0.5], [1.0])
    with pytest.raises(ValueError):
        prl.error_norm(prl.NormKind.L2, [], [])


def test_from_csr_roundtrip_and_validation(prl, oracle):
    n, pairs = oracle.rmat(12, 16, 0.57, 0.19, 0.19, 9)
    want = oracle.build_csr(n, pairs)
    g = prl.csr_from_arrays(n, want.in_offsets, want.in_neighbors, want.out_degree)
    assert np.array_equal(g.in_offsets, want.in_offsets)
    assert np.array_equal(g.in_neighbors, want.in_neighbors)
    assert np.array_equal(g.dangling, want.dangling)
    with pytest.raises(ValueError):
        prl.build_csr(prl.EdgeList(3, np.array([[0, 5]], np.uint32)))
    with pytest.raises(ValueError):  # in-neighbour out of range
        prl.csr_from_arrays(3, np.array([0, 1, 1, 1], np.uint64), np.array([7], np.uint32),
                            np.array([1, 0, 0], np.uint32))
    with pytest.raises(ValueError):  # in-neighbour with out_degree 0: pagerank.hpp:91 divides by it
        prl.csr_from_arrays(3, np.array([0, 1, 1, 1], np.uint64), np.array([2], np.uint32),
                            np.array([1, 0, 0], np.uint32))


def test_from_csr_hand_filled_like_reference(prl, ref):
    """A hand-filled CsrGraph (graph.hpp:47-60) is used by pagerank() as given
    (pagerank.hpp:89-93): rows in any order, duplicate in-neighbours counted
    twice, out_degree taken from the caller even where it differs from the
    neighbour histogram.  The device graph accepts the same arrays and the
    run matches the reference's own pagerank on them."""
    rs = np.random.default_rng(7)
    n = 3000
    rows = []
    for v in range(n):
        d = int(rs.integers(0, 12)) if v % 17 else int(rs.integers(200, 5000))  # some hub rows
        rows.append(rs.integers(0, n, d).astype(np.uint32))  # unsorted, with duplicates
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(r) for r in rows])
    nbr = np.concatenate(rows).astype(np.uint32)
    hist = np.bincount(nbr, minlength=n).astype(np.uint32)
    deg = hist + (rs.integers(0, 3, n) * (hist > 0)).astype(np.uint32)  # inflated degrees
    deg[(hist == 0) & (rs.random(n) < 0.3)] = 5  # sources the graph never gathers
    assert np.any(np.diff(nbr.astype(np.int64)) < 0) and len(np.unique(nbr)) < nbr.size
    g = prl.csr_from_arrays(n, off, nbr, deg)
    assert np.array_equal(g.out_degree, deg)
    h = ref.csr_from_arrays(n, off, nbr, deg)
    try:
        for a, norm in ((0.85, "l1"), (0.95, "l2"), (1.0, "linf")):
            want = ref.pagerank(h, a, 1e-10, norm, 500, trace=True)
            got = prl.pagerank(g, prl.PageRankConfig(a, 1e-10, nk(prl, norm), 500))
            assert iterations_match(got.iterations, want["iterations"], want["err_trace"], 1e-10), a
            assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, a
    finally:
        ref.free_csr(h)


def test_from_csr_sliced_build_matches_generator(prl):
    """graph_from_csr uploads the neighbour array in 8M-edge slices and sorts
    each slice's complete rows while later slices are in flight; the
    generator builds the same graph in one piece and sorts rows per length
    band.  Same engine layout => bit-identical runs (the kernels are
    deterministic and a row's summation order is its source order)."""
    g1 = prl.generate_rmat(20, 16, 0.57, 0.19, 0.19, 2108)
    assert g1.edge_count() > 2 * (8 << 20) - (1 << 20)  # two or more slices
    g2 = prl.csr_from_arrays(g1.vertex_count, g1.in_offsets, g1.in_neighbors, g1.out_degree)
    a = prl.pagerank_batched(g1, [0.5, 0.85, 1.0], 1e-9, prl.NormKind.L1, 200)
    b = prl.pagerank_batched(g2, [0.5, 0.85, 1.0], 1e-9, prl.NormKind.L1, 200)
    for k in range(3):
        assert a.results[k].iterations == b.results[k].iterations
        assert np.array_equal(a.results[k].ranks, b.results[k].ranks), k


# ---------------------------------------------------------------------------
# Benchmark configs (BASELINE.json) — device generators, then parity
# ---------------------------------------------------------------------------
def graph_hashes(oracle, g):
    return dict(h_offsets=oracle.hash64(g.in_offsets), h_neighbors=oracle.hash64(g.in_neighbors),
                h_degree=oracle.hash64(g.out_degree), h_dangling=oracle.hash64(g.dangling))


def test_c1_rmat16(prl, oracle):
    gold = load_golden("c1_rmat16.json")
    arr = np.load(os.path.join(GOLD, "c1_rmat16.npz"))
    g = prl.generate_rmat(16, 16, 0.57, 0.19, 0.19, gold["seed"])
    assert g.vertex_count == gold["graph"]["n"] and g.edge_count() == gold["graph"]["e"]
    for k, v in graph_hashes(oracle, g).items():
        assert v == gold["graph"][k], k
    # host-generated pairs through build_csr agree too
    n, pairs = oracle.rmat(16, 16, 0.57, 0.19, 0.19, gold["seed"])
    g2 = prl.build_csr(edge_list(prl, n, pairs))
    assert graph_hashes(oracle, g2) == graph_hashes(oracle, g)
    for norm in NORMS:
        r = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-6, nk(prl, norm)))
        tr = arr[f"trace_{norm}"]
        assert iterations_match(r.iterations, gold["runs"][norm]["iterations"], tr, 1e-6), norm
        assert np.max(np.abs(r.ranks - arr[f"ranks_{norm}"])) <= RANK_TOL


def test_c1_determinism_and_batched_lanes(prl):
    g = prl.generate_rmat(16, 16, 0.57, 0.19, 0.19, 2108)
    a = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-8))
    b = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-8))
    assert np.array_equal(a.ranks, b.ranks) and a.iterations == b.iterations
    alphas = [0.5, 0.6, 0.75, 0.85, 0.95]
    br = prl.pagerank_batched(g, alphas, 1e-8)
    for k, al in enumerate(alphas):
        one = prl.pagerank(g, prl.PageRankConfig(al, 1e-8))
        assert br.results[k].iterations == one.iterations
        assert np.max(np.abs(br.results[k].ranks - one.ranks)) <= 1e-13


def test_c2_rmat22_damping_sweep(prl, oracle):
    gold = load_golden("c2_rmat22.json")
    arr = np.load(os.path.join(GOLD, "c2_rmat22.npz"))
    g = prl.generate_rmat(22, 16, 0.57, 0.19, 0.19, gold["seed"])
    assert g.edge_count() == gold["graph"]["e"]
    for k, v in graph_hashes(oracle, g).items():
        assert v == gold["graph"][k], k
    alphas = [ln["alpha"] for ln in gold["lanes"]]
    ref = prl.reference_ranks(g)
    br = prl.pagerank_batched(g, alphas, 1e-6, prl.NormKind.L1, 500, ref_ranks=ref)
    idx = arr["sample_idx"]
    for k, ln in enumerate(gold["lanes"]):
        r = br.results[k]
        assert iterations_match(r.iterations, ln["iterations"], arr[f"lane{k}_trace"], 1e-6), k
        assert r.converged == ln["converged"]
        assert np.max(np.abs(r.ranks[idx] - arr[f"lane{k}_sample"])) <= RANK_TOL
        assert np.max(np.abs(r.ranks[arr[f"lane{k}_top_idx"]] - arr[f"lane{k}_top"])) <= RANK_TOL
        assert abs(float(np.sum(r.ranks.astype(np.longdouble))) - float(arr[f"lane{k}_total"])) <= 1e-9
        err = float(br.trace[r.iterations - 1, k, 3])
        assert math.isclose(err, ln["err_vs_ref"], rel_tol=1e-6, abs_tol=1e-12), k


def test_c3_grid_tolerance_norm_sweep(prl, oracle):
    path = os.path.join(GOLD, "c3_grid4096.json")
    if not os.path.exists(path):
        pytest.skip("c3 golden not generated")
    gold = load_golden("c3_grid4096.json")
    arr = np.load(os.path.join(GOLD, "c3_grid4096.npz"))
    g = prl.generate_grid(4096, 0.6, 0.01, gold["seed"])
    assert g.edge_count() == gold["graph"]["e"]
    for k, v in graph_hashes(oracle, g).items():
        assert v == gold["graph"][k], k
    taus = [10.0 ** -k for k in range(1, 11)]
    plan = prl.SweepPlan(graphs=["grid4096"], alphas=[0.85], tolerances=taus,
                         norms=list(prl.all_norms), repeats=1)
    recs = prl.run_sweep(plan, graphs_override={"grid4096": g})
    assert len(recs) == 30
    want = {(c["norm"], c["tol"]): c for c in gold["cells"]}
    for rec in recs:
        c = want[(prl.norm_name(rec.norm), rec.tolerance)]
        tr = arr[f"trace_{prl.norm_name(rec.norm)}"]
        assert iterations_match(rec.iterations, c["iterations"], tr, rec.tolerance), c
        assert rec.converged == c["converged"]
        assert math.isclose(rec.err_vs_ref, c["err_vs_ref"], rel_tol=1e-6, abs_tol=1e-13), c
    # final ranks of the tightest cell per norm
    idx = arr["sample_idx"]
    for norm in NORMS:
        r = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-10, nk(prl, norm)))
        assert r.iterations == gold["runs"][norm]["iterations"]
        assert np.max(np.abs(r.ranks[idx] - arr[f"{norm}_final_sample"])) <= RANK_TOL


def test_c4_rmat26_linf(prl, oracle):
    """configs[3]: RMAT-26 (67M vertices, 1.06B edges), alpha .85, tau 1e-10,
    Linf — graph fingerprint bit-exact, iteration count, sampled/top/total ranks."""
    gold = load_golden("c4_rmat26.json")
    arr = np.load(os.path.join(GOLD, "c4_rmat26.npz"))
    g = prl.generate_rmat(26, 16, 0.57, 0.19, 0.19, gold["seed"])
    assert g.edge_count() == gold["graph"]["e"]
    for k, v in graph_hashes(oracle, g).items():
        assert v == gold["graph"][k], k
    r = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-10, prl.NormKind.LInf))
    assert iterations_match(r.iterations, gold["iterations"], arr["trace"], 1e-10)
    assert r.converged == gold["converged"]
    idx = arr["sample_idx"]
    assert np.max(np.abs(r.ranks[idx] - arr["sample"])) <= RANK_TOL
    assert np.max(np.abs(r.ranks[arr["top_idx"]] - arr["top"])) <= RANK_TOL
    assert abs(float(np.sum(r.ranks.astype(np.longdouble))) - float(arr["total"])) <= 1e-9


@pytest.mark.parametrize("K", [2, 3, 5, 8, 9, 12, 13, 16])
def test_batched_lane_modes_vs_oracle(prl, oracle, K):
    """Batched runs of every lane-width family, lanes freezing in an order the
    slowest-first storage does not predict (per-lane tolerances), so the run
    walks through the narrow modes and their repacks; every lane must match
    the oracle's single run: iterations (+-1 rule) and ranks <= 1e-10."""
    rng = np.random.default_rng(1000 + K)
    n, pairs = oracle.rmat(14, 16, 0.57, 0.19, 0.19, 77)
    h = oracle.build_csr_handle(n, pairs)
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 77)
    alphas = list(np.round(rng.uniform(0.3, 0.99, K), 3))
    tols = 10.0 ** -rng.uniform(4, 10, K)
    br = prl.pagerank_batched(g, alphas, tols, prl.NormKind.L1, 500)
    for k in range(K):
        want = oracle.pagerank(h, alphas[k], tols[k], "l1", 500, trace=True)
        got = br.results[k]
        assert iterations_match(got.iterations, want["iterations"], want["err_trace"], tols[k]), k
        assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, k
    oracle.free_csr(h)


def test_graph_rows_matches_download(prl):
    """prgpu_graph_rows (row-sample download for graphs too large to pull back
    whole) agrees with the full reference-layout download."""
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 31)
    n = g.vertex_count
    rows = np.array([0, 5, n - 1] + list(range(100, n, 97)), np.uint32)
    off, nbr = g.rows(rows)
    full_off, full_nbr = g.in_offsets, g.in_neighbors
    want = [full_nbr[full_off[v]:full_off[v + 1]] for v in rows]
    assert np.array_equal(np.diff(off), [len(w) for w in want])
    assert np.array_equal(nbr, np.concatenate(want))
    assert np.array_equal(g.out_degree_only(), g.out_degree)
    with pytest.raises(ValueError):
        g.rows([n])


def test_load_csr_graph_mtx(prl, ref, tmp_path):
    """load_csr_graph (graph.hpp:249-251): parallel MatrixMarket parse +
    device build_csr, CSR identical to the reference's on a symmetric,
    weighted file with comments."""
    rng = np.random.default_rng(7)
    n, m = 3000, 20000
    r, c = rng.integers(1, n + 1, m), rng.integers(1, n + 1, m)
    path = tmp_path / "g.mtx"
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n% test\n")
        f.write(f"{n} {n} {m}\n")
        for i in range(m):
            f.write(f"{r[i]} {c[i]} {rng.random():.6f}\n")
    g = prl.load_csr_graph(path)
    rn, rp = ref.load_mtx(str(path))
    want = ref.build_csr(rn, rp.reshape(-1))
    for key in ("in_offsets", "in_neighbors", "out_degree", "dangling"):
        assert np.array_equal(getattr(g, key), getattr(want, key)), key
    with pytest.raises(RuntimeError, match="cannot open graph file"):
        prl.load_csr_graph(tmp_path / "none.mtx")


def test_concurrent_pagerank_on_shared_graph(prl):
    """SPEC.md:194 / sweep.hpp:209-225: pagerank is reentrant on a shared,
    immutable graph.  Host threads (ctypes drops the GIL) solve different
    configs on one graph at once, plus builds of other graphs; every result
    equals the same call made alone, bit for bit."""
    import threading
    g = prl.generate_rmat(16, 16, 0.57, 0.19, 0.19, 2108)
    cfgs = [prl.PageRankConfig(a, t, nm) for a in (0.6, 0.85, 0.95)
            for t, nm in ((1e-6, prl.NormKind.L1), (1e-9, prl.NormKind.L2), (1e-8, prl.NormKind.LInf))]
    alone = [prl.pagerank(g, c) for c in cfgs]
    out = [None] * len(cfgs)
    built = [None] * 4
    errors = []

    def solve(i):
        try:
            out[i] = prl.pagerank(g, cfgs[i])
        except Exception as e:  # surfaced below
            errors.append(e)

    def build(i):
        try:
            built[i] = prl.generate_rmat(12, 16, 0.57, 0.19, 0.19, 100 + i).edge_count()
        except Exception as e:
            errors.append(e)

    ts = [threading.Thread(target=solve, args=(i,)) for i in range(len(cfgs))]
    ts += [threading.Thread(target=build, args=(i,)) for i in range(len(built))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for a, b in zip(alone, out):
        assert a.iterations == b.iterations and np.array_equal(a.ranks, b.ranks)
    for i in range(len(built)):
        assert built[i] == prl.generate_rmat(12, 16, 0.57, 0.19, 0.19, 100 + i).edge_count()


def test_acceptance_sensitivity_and_damping_trend(prl, oracle, small_golden):
    """acceptance.cpp:261-329 through the product API on the 10k scale-free
    fixture (seed 2021): at alpha .95 over the tolerance grid extended to
    1e-16, L1 hits the sensitivity limit and no later than L2 / LInf, and
    each norm's failing tail is exactly its non-converged cells; the
    iteration ratios 0.95/0.85 in [2, 4] and 0.75/0.85 in [0.4, 0.8] equal
    the reference's iteration counts."""
    sf = small_golden["known"]["scale_free_10k"]
    rng = oracle.mt19937(2021)
    n, pairs = oracle.scale_free_web(rng, 10000, 4, 0.08)
    g = prl.build_csr(edge_list(prl, n, pairs))
    grid = list(prl.default_tolerance_grid()) + [5e-11, 1e-11, 5e-12, 1e-12, 5e-13, 1e-13,
                                                 5e-14, 1e-14, 5e-15, 1e-15, 5e-16, 1e-16]
    recs = []
    for norm in prl.all_norms:
        for tol in grid:
            r = prl.pagerank(g, prl.PageRankConfig(0.95, tol, norm))
            recs.append(prl.SweepRecord("scale_free_10k", n, g.edge_count(), 0.95, tol, norm,
                                        r.iterations, r.converged))
    first = {int(f.norm): f.first_failing_tolerance for f in prl.detect_sensitivity(recs)}
    l1, l2, linf = (first[int(k)] for k in (prl.NormKind.L1, prl.NormKind.L2, prl.NormKind.LInf))
    assert l1 is not None
    if l2 is not None:
        assert l1 >= l2
    if linf is not None:
        assert l1 >= linf
    for rec in recs:
        f = first[int(rec.norm)]
        in_tail = f is not None and rec.tolerance <= f
        assert rec.converged == (not in_tail), (rec.norm, rec.tolerance)
    its = {a: prl.pagerank(g, prl.PageRankConfig(a, 1e-6, prl.NormKind.L1)).iterations
           for a in (0.75, 0.85, 0.95)}
    for a, it in its.items():
        assert it == sf["damping"][f"{a:.2f}"], (a, it)
    assert 2.0 <= its[0.95] / its[0.85] <= 4.0 and 0.4 <= its[0.75] / its[0.85] <= 0.8


def _structural_graphs():
    """Shapes that stress the task decomposition: one huge hub row (chunk
    hand-off), one huge source, chains, isolated vertices, no edges, dense
    rows, rows exactly at the chunk/packed thresholds, self-loops."""
    rng = np.random.default_rng(99)
    out = {}
    n = 300_001
    src = np.arange(1, n, dtype=np.uint32)
    out["big_star_in"] = (n, np.concatenate([np.stack([src, np.zeros_like(src)], 1), [[0, 1]]]))
    out["big_star_out"] = (n, np.stack([np.zeros_like(src), src], 1))
    m = 100_000
    a = np.arange(m - 1, dtype=np.uint32)
    out["chain"] = (m, np.stack([a, a + 1], 1))
    out["one_edge"] = (1000, np.array([[5, 7]], np.uint32))
    out["no_edges"] = (10, np.zeros((0, 2), np.uint32))
    k = 50
    ii, jj = np.meshgrid(np.arange(k), np.arange(k))
    msk = ii != jj
    out["complete_50"] = (k, np.stack([ii[msk], jj[msk]], 1).astype(np.uint32))
    # target t gets exactly d in-edges from distinct sources, d at the thresholds
    degs = [1, 8, 9, 32, 33, 128, 129, 256, 257, 512, 513, 2048, 2049, 4096, 4097, 8193]
    nn = 20_000
    pairs = []
    for t, d in enumerate(degs):
        s = rng.choice(np.arange(len(degs), nn), size=d, replace=False)
        pairs.append(np.stack([s, np.full(d, t)], 1))
    extra = rng.integers(0, nn, size=(40_000, 2))
    out["thresholds"] = (nn, np.concatenate(pairs + [extra]).astype(np.uint32))
    nl = 5000
    loops = np.arange(nl, dtype=np.uint32)
    out["self_loops"] = (nl, np.concatenate([np.stack([loops, loops], 1),
                                             rng.integers(0, nl, size=(20_000, 2)).astype(np.uint32)]))
    return out


@pytest.mark.parametrize("name", ["big_star_in", "big_star_out", "chain", "one_edge", "no_edges",
                                  "complete_50", "thresholds", "self_loops"])
def test_structural_edge_cases_vs_oracle(prl, oracle, name):
    n, pairs = _structural_graphs()[name]
    flat = np.ascontiguousarray(pairs, np.uint32).reshape(-1)
    g = prl.build_csr(edge_list(prl, n, flat))
    want_g = oracle.build_csr(n, flat)
    assert np.array_equal(g.in_offsets, want_g.in_offsets) and np.array_equal(g.in_neighbors, want_g.in_neighbors)
    h = oracle.build_csr_handle(n, flat)
    try:
        for norm in NORMS:  # K = 1, every norm
            want = oracle.pagerank(h, 0.85, 1e-10, norm, 500, trace=True)
            got = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-10, nk(prl, norm), 500))
            assert iterations_match(got.iterations, want["iterations"], want["err_trace"], 1e-10), (norm,)
            assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, norm
        alphas = [0.5, 0.85, 1.0]  # batched lanes (lane-width modes switch as they stop)
        br = prl.pagerank_batched(g, alphas, 1e-9, prl.NormKind.L1, 300)
        for k, a in enumerate(alphas):
            want = oracle.pagerank(h, a, 1e-9, "l1", 300, trace=True)
            r = br.results[k]
            assert iterations_match(r.iterations, want["iterations"], want["err_trace"], 1e-9), (a,)
            assert np.max(np.abs(r.ranks - want["ranks"])) <= RANK_TOL, a
    finally:
        oracle.free_csr(h)


@pytest.mark.parametrize("K,keep", [(1, None), (3, None), (11, None), (3, "0"), (11, "0")])
def test_series_sweep_vs_oracle(prl, oracle, K, keep, monkeypatch):
    """The power-series sweep (one alpha = 1 chain, per-lane weighted sums)
    against the oracle's separate runs: iterations (+-1 rule), converged,
    ranks <= 1e-10, and the err traces to the reference's rounding noise;
    alpha 0 and 1 included; per-lane tolerances and all-norm stop masks.
    keep "0" forces the large-graph variant (sums accumulated as the chain
    runs) that C5 uses."""
    if keep is not None:
        monkeypatch.setenv("PRGPU_SERIES_KEEP", keep)
    rng = np.random.default_rng(500 + K)
    n, pairs = oracle.rmat(14, 16, 0.57, 0.19, 0.19, 77)
    h = oracle.build_csr_handle(n, pairs)
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 77)
    try:
        alphas = [0.0, 1.0, 0.85][:K] if K <= 3 else list(np.round(rng.uniform(0.3, 1.0, K), 3))
        tols = list(10.0 ** -rng.uniform(4, 10, K))
        for norm, mask in ((prl.NormKind.L1, 0), (prl.NormKind.L2, 0), (prl.NormKind.LInf, 7)):
            br = prl.pagerank_batched(g, alphas, tols, norm, 500, stop_mask=mask, series=True)
            for k in range(K):
                got = br.results[k]
                names = ["l1", "l2", "linf"]
                if mask == 7:  # every norm must be below tau: the latest crossing of the three
                    runs = [oracle.pagerank(h, alphas[k], tols[k], nm, 500, trace=True) for nm in names]
                    want = max(runs, key=lambda r: r["iterations"])
                    tr = want["err_trace"]
                else:
                    want = oracle.pagerank(h, alphas[k], tols[k], names[int(norm)], 500, trace=True)
                    tr = want["err_trace"]
                assert iterations_match(got.iterations, want["iterations"], tr, tols[k]), (k, norm)
                assert got.converged == want["converged"]
                assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, (k, norm)
            # traces: lane k's err at every iteration it ran, under the run's norm
            if mask == 0:
                for k in range(K):
                    want = oracle.pagerank(h, alphas[k], tols[k], ["l1", "l2", "linf"][int(norm)], 500, trace=True)
                    m = min(br.results[k].iterations, len(want["err_trace"]))
                    got_tr = br.trace[:m, k, int(norm)]
                    ref_tr = np.asarray(want["err_trace"][:m])
                    # the reference differences two iterates of size ~1/N each: its err
                    # carries ~1e-13 of rounding noise (the series computes
                    # alpha^t * ||y_t - y_{t-1}||, equal in exact arithmetic)
                    assert np.allclose(got_tr, ref_tr, rtol=1e-6, atol=1e-13), k
    finally:
        oracle.free_csr(h)


@pytest.mark.parametrize("keep", ["1", "0"])
def test_series_capped_matches_batched(prl, keep, monkeypatch):
    """Iteration caps 1, 2, 3 and 7 (the chain's lookahead must never run a
    lane past its cap): the series and the batched run agree on iterations,
    converged flags, final errors and ranks."""
    monkeypatch.setenv("PRGPU_SERIES_KEEP", keep)
    g = prl.generate_rmat(13, 8, 0.57, 0.19, 0.19, 31)
    alphas = [0.3, 0.85, 0.99]
    for cap in (1, 2, 3, 7):
        a = prl.pagerank_batched(g, alphas, 1e-12, prl.NormKind.L2, cap)
        b = prl.pagerank_batched(g, alphas, 1e-12, prl.NormKind.L2, cap, series=True)
        for k in range(3):
            assert b.results[k].iterations == a.results[k].iterations == cap, (cap, k)
            assert b.results[k].converged == a.results[k].converged
            assert abs(b.results[k].final_err - a.results[k].final_err) <= 1e-6 * a.results[k].final_err + 1e-16
            assert np.max(np.abs(b.results[k].ranks - a.results[k].ranks)) <= 1e-13, (cap, k)


def test_series_sweep_c2_golden(prl):
    """C2 (RMAT-22, 11 alphas) through the series sweep against the reference's
    goldens: iterations per lane, converged, sampled and top ranks, rank sums."""
    gold = load_golden("c2_rmat22.json")
    arr = np.load(os.path.join(GOLD, "c2_rmat22.npz"))
    g = prl.generate_rmat(22, 16, 0.57, 0.19, 0.19, gold["seed"])
    alphas = [ln["alpha"] for ln in gold["lanes"]]
    br = prl.pagerank_batched(g, alphas, 1e-6, prl.NormKind.L1, 500, series=True)
    idx = arr["sample_idx"]
    for k, ln in enumerate(gold["lanes"]):
        r = br.results[k]
        assert iterations_match(r.iterations, ln["iterations"], arr[f"lane{k}_trace"], 1e-6), k
        assert r.converged == ln["converged"]
        assert np.max(np.abs(r.ranks[idx] - arr[f"lane{k}_sample"])) <= RANK_TOL
        assert np.max(np.abs(r.ranks[arr[f"lane{k}_top_idx"]] - arr[f"lane{k}_top"])) <= RANK_TOL
        assert abs(float(np.sum(r.ranks.astype(np.longdouble))) - float(arr[f"lane{k}_total"])) <= 1e-9


EXP_LIB = "libprgpu_exp.so"  # make -C paper_2108_02997_b200/csrc EXPERIMENTS=1


@pytest.mark.skipif(not os.environ.get("PRGPU_LIB", "").endswith(EXP_LIB),
                    reason="the split pull is compiled into the tuning build only (tests/test_experiments_gpu.py)")
@pytest.mark.parametrize("split_mb", ["1", "4"])
def test_split_pull_matches_oracle(prl, oracle, monkeypatch, split_mb):
    """The split pull (PRGPU_SPLIT_MB: hot-source CSR pass, then cold-source
    pass adding the hot partial) against the oracle: exact iterations, ranks
    within 1e-10, for one and several lanes and every norm; and against the
    one-pass run (same iterations, ranks to rounding)."""
    n, pairs = oracle.rmat(17, 16, 0.57, 0.19, 0.19, 2108)
    h = oracle.build_csr_handle(n, pairs)
    g = prl.build_csr(edge_list(prl, n, pairs))
    try:
        one = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        monkeypatch.setenv("PRGPU_SPLIT_MB", split_mb)
        for norm in ("l1", "l2", "linf"):
            want = oracle.pagerank(h, 0.85, 1e-9, norm, 300)
            got = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-9, nk(prl, norm), 300))
            assert got.iterations == want["iterations"], norm
            assert np.max(np.abs(got.ranks - want["ranks"])) <= RANK_TOL, norm
        two = prl.pagerank_batched(g, [0.95, 0.85, 0.6], 1e-9, prl.NormKind.L2, 300)
        for a, b, alpha in zip(one.results, two.results, (0.95, 0.85, 0.6)):
            assert a.iterations == b.iterations
            assert np.max(np.abs(a.ranks - b.ranks)) <= 1e-15
            want = oracle.pagerank(h, alpha, 1e-9, "l2", 300)
            assert b.iterations == want["iterations"]
            assert np.max(np.abs(b.ranks - want["ranks"])) <= RANK_TOL
        eleven = [0.5 + 0.05 * i for i in range(11)]
        w = prl.pagerank_batched(g, eleven, 1e-6, prl.NormKind.L1, 300)
        monkeypatch.delenv("PRGPU_SPLIT_MB")
        u = prl.pagerank_batched(g, eleven, 1e-6, prl.NormKind.L1, 300)
        for a, b in zip(w.results, u.results):
            assert a.iterations == b.iterations and np.max(np.abs(a.ranks - b.ranks)) <= 1e-15
    finally:
        oracle.free_csr(h)


def test_error_norm_device_vs_reference_long_double(prl, ref):
    """prgpu_error_norm carries L1 / L2 sums as double-double (the reference
    accumulates in x87 long double, norms.hpp:57-69): equal to the
    reference's result to within one double ulp on rank-like vectors of
    1e3..4e6 entries (the reference's own long-double rounding), Linf exactly."""
    rs = np.random.default_rng(2021)
    for n in (1000, 100_000, 4_000_000):
        r = rs.random(n) / n
        s = r + (rs.random(n) - 0.5) * 1e-7 / n
        s[rs.integers(0, n, 10)] += 1e-3 / n  # a few outliers
        for norm, kind in (("l1", prl.NormKind.L1), ("l2", prl.NormKind.L2), ("linf", prl.NormKind.LInf)):
            want = ref.error_norm(norm, r, s)
            got = prl.error_norm(kind, r, s)
            if norm == "linf":
                assert got == want
            else:
                assert abs(got - want) <= np.spacing(want), (n, norm, got, want)
