"""CPU: the oracle restatement (oracle/oracle.c) pinned against the reference.

Pins: tests/golden/*.json (written from the reference itself by
oracle/make_goldens.py) and, where oracle/_ref is built, the reference's own
build_csr / pagerank / error_norm / generators called side by side.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, load_golden

NORMS = ["l1", "l2", "linf"]


def test_fixture_csr_and_runs_bit_exact(oracle, small_golden):
    for name, fx in small_golden["fixtures"].items():
        pairs = np.array(fx["pairs"], np.uint32)
        g = oracle.build_csr(fx["n"], pairs)
        for key in ("in_offsets", "in_neighbors", "out_degree", "dangling"):
            assert getattr(g, key).tolist() == fx["csr"][key], (name, key)
        h = oracle.build_csr_handle(fx["n"], pairs)
        for run in fx["runs"]:
            got = oracle.pagerank(h, run["alpha"], run["tol"], run["norm"], run["max_iter"],
                                  trace=True)
            assert got["iterations"] == run["iterations"], (name, run["alpha"], run["norm"])
            assert got["converged"] == run["converged"]
            assert got["ranks"].tolist() == run["ranks"]          # bit-exact
            assert got["err_trace"].tolist() == run["err_trace"]  # bit-exact
        oracle.free_csr(h)


def test_acceptance_trials_bit_exact(oracle, small_golden):
    """acceptance.cpp:104-132 trial set: restatement == reference, bit for bit,
    and the dense oracle agrees (identical iterations, Linf <= 1e-8)."""
    for t in small_golden["trials"]:
        pairs = np.array(t["pairs"], np.uint32)
        h = oracle.build_csr_handle(t["n"], pairs)
        got = oracle.pagerank(h, t["alpha"], t["tol"], t["norm"], 500, trace=True)
        oracle.free_csr(h)
        assert got["iterations"] == t["iterations"]
        assert got["ranks"].tolist() == t["ranks"]
        dense = oracle.dense_pagerank(t["n"], pairs, t["alpha"], t["tol"], t["norm"])
        assert dense["iterations"] == t["dense_iterations"] == t["iterations"]
        assert np.max(np.abs(dense["ranks"] - np.array(t["ranks"]))) <= 1e-8


def test_known_answers(oracle, small_golden):
    k = small_golden["known"]
    for a, tol, want in k["estimates"]:
        assert oracle.estimate_iterations(a, tol) == want
    for bad in [(1.0, 1e-6), (0.0, 1e-6), (0.85, 1.0), (0.85, 0.0)]:
        with pytest.raises(ValueError):
            oracle.estimate_iterations(*bad)
    n, pairs = oracle.regular_ring(1000, 3)
    h = oracle.build_csr_handle(n, pairs)
    for norm, tol, it in k["ring_1000_3"]:
        assert oracle.pagerank(h, 0.85, tol, norm)["iterations"] == it == 1
    oracle.free_csr(h)
    # star closed form (test_pagerank.cpp:34-38,69-87)
    h = oracle.build_csr_handle(3, np.array([1, 0, 2, 0], np.uint32))
    r = oracle.pagerank(h, 0.85, 1e-10, "l1")
    c = 1.0 / (3.0 + 2 * 0.85)
    assert np.allclose(r["ranks"], [(1 + 2 * 0.85) * c, c, c], rtol=1e-6)
    oracle.free_csr(h)


def test_scale_free_damping_and_sensitivity(oracle, small_golden):
    sf = small_golden["known"]["scale_free_10k"]
    rng = oracle.mt19937(2021)
    n, pairs = oracle.scale_free_web(rng, 10000, 4, 0.08)
    assert n == sf["n"] and pairs.size // 2 == sf["m"]
    h = oracle.build_csr_handle(n, pairs)
    for a, it in sf["damping"].items():
        assert oracle.pagerank(h, float(a), 1e-6, "l1")["iterations"] == it
    up = sf["damping"]["0.95"] / sf["damping"]["0.85"]
    down = sf["damping"]["0.75"] / sf["damping"]["0.85"]
    assert 2.0 <= up <= 4.0 and 0.4 <= down <= 0.8  # acceptance.cpp:314-329
    for tr in sf["sensitivity_alpha095"]["traces"]:
        got = oracle.pagerank(h, 0.95, 1e-300, tr["norm"], 500, trace=True)
        assert got["err_trace"].tolist() == tr["err_trace"]
    r = oracle.pagerank(h, 0.85, 1e-6, "l1")
    assert r["ranks"].tolist() == sf["ranks_085"]
    oracle.free_csr(h)


def test_norm_hand_values(oracle):
    # test_norms.cpp:17-24
    r, s = np.array([0.3, 0.7]), np.array([0.5, 0.5])
    assert abs(oracle.error_norm("l1", r, s) - 0.4) < 1e-12
    assert abs(oracle.error_norm("linf", r, s) - 0.2) < 1e-12
    assert abs(oracle.error_norm("l2", r, s) - np.sqrt(0.08)) < 1e-12
    for k in NORMS:
        assert oracle.error_norm(k, r, r) == 0.0


def test_c1_golden(oracle):
    gold = load_golden("c1_rmat16.json")
    arr = np.load(os.path.join(GOLD, "c1_rmat16.npz"))
    n, pairs = oracle.rmat(16, 16, 0.57, 0.19, 0.19, gold["seed"])
    assert oracle.hash64(pairs) == gold["graph"]["h_pairs"]
    g = oracle.build_csr(n, pairs)
    assert oracle.hash64(g.in_offsets) == gold["graph"]["h_offsets"]
    assert oracle.hash64(g.in_neighbors) == gold["graph"]["h_neighbors"]
    assert oracle.hash64(g.out_degree) == gold["graph"]["h_degree"]
    assert oracle.hash64(g.dangling) == gold["graph"]["h_dangling"]
    h = oracle.build_csr_handle(n, pairs)
    for norm in NORMS:
        r = oracle.pagerank(h, 0.85, 1e-6, norm, trace=True)
        assert r["iterations"] == gold["runs"][norm]["iterations"]
        assert np.array_equal(r["ranks"], arr[f"ranks_{norm}"])
        assert np.array_equal(r["err_trace"], arr[f"trace_{norm}"])
    oracle.free_csr(h)


@pytest.mark.parametrize("name,scale_or_side", [("c2_rmat22.json", 22), ("c3_grid4096.json", 4096)])
def test_large_generator_pins(oracle, name, scale_or_side):
    """The benchmark generators reproduce the graphs the goldens were made on
    (hash of the raw edge list; CSR hashes are checked in the GPU tests)."""
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    gold = load_golden(name)
    if name.startswith("c2"):
        n, pairs = oracle.rmat(22, 16, 0.57, 0.19, 0.19, gold["seed"])
    else:
        n, pairs = oracle.grid(4096, 0.6, 0.01, gold["seed"])
    assert n == gold["graph"]["n"]
    assert pairs.size // 2 == gold["graph"]["raw_edges"]
    assert oracle.hash64(pairs) == gold["graph"]["h_pairs"]


def test_restatement_matches_reference_live(oracle, ref):
    """Side by side with the reference's own code on fresh random inputs."""
    o_rng, r_rng = oracle.mt19937(77), ref.rng(77)
    for trial in range(30):
        n = 2 + trial
        a = oracle.random_digraph(o_rng, n, 0.2, trial % 2 == 0)
        b = ref.random_digraph(r_rng, n, 0.2, trial % 2 == 0)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
    ref.rng_free(r_rng)
    n, pairs = oracle.rmat(12, 16, 0.57, 0.19, 0.19, 5)
    go, gr = oracle.build_csr(n, pairs), ref.build_csr(n, pairs)
    for key in ("in_offsets", "in_neighbors", "out_degree", "dangling"):
        assert np.array_equal(getattr(go, key), getattr(gr, key))
    ho, hr = oracle.build_csr_handle(n, pairs), ref.build_csr_handle(n, pairs)
    for norm in NORMS:
        for alpha in (0.0, 0.6, 1.0):
            x = oracle.pagerank(ho, alpha, 1e-9, norm, trace=True)
            y = ref.pagerank(hr, alpha, 1e-9, norm, trace=True)
            assert x["iterations"] == y["iterations"]
            assert np.array_equal(x["ranks"], y["ranks"])
            assert np.array_equal(x["err_trace"], y["err_trace"])
    rs = np.random.default_rng(3).random((2, 100))
    for norm in NORMS:
        assert oracle.error_norm(norm, rs[0], rs[1]) == ref.error_norm(norm, rs[0], rs[1])
    oracle.free_csr(ho)
    ref.free_csr(hr)


def test_step_rows_is_one_reference_iteration(oracle):
    """orc_pagerank_step_rows (the C5 one-step checker) reproduces iteration t
    of the full restatement bit for bit from iteration t-1, on every row and on
    a row subset (reference layout, ascending neighbours)."""
    n, pairs = oracle.rmat(14, 16, 0.57, 0.19, 0.19, 9)
    g = oracle.build_csr(n, pairs)
    h = oracle.build_csr_handle(n, pairs)
    for alpha in (0.5, 0.85, 1.0):
        for t in (1, 2, 5):
            prev = oracle.pagerank(h, alpha, 1e-30, "l1", max_iter=t - 1)["ranks"] if t > 1 \
                else np.full(n, 1.0 / n)
            nxt = oracle.pagerank(h, alpha, 1e-30, "l1", max_iter=t)["ranks"]
            got, c0 = oracle.step_rows(prev, g.out_degree, alpha, g.in_offsets, g.in_neighbors)
            assert np.array_equal(got, nxt), (alpha, t)
            rows = np.arange(0, n, 37, dtype=np.uint32)
            off = np.zeros(len(rows) + 1, np.uint64)
            off[1:] = np.cumsum(g.in_offsets[rows + 1] - g.in_offsets[rows])
            nbr = np.concatenate([g.in_neighbors[g.in_offsets[v]:g.in_offsets[v + 1]] for v in rows])
            sub, _ = oracle.step_rows(prev, g.out_degree, alpha, off, nbr)
            assert np.array_equal(sub, nxt[rows])
    oracle.free_csr(h)


def test_pagerank_mt_bit_identical(oracle, ref):
    """orc_pagerank_mt (the vertex loop on host threads, the CPU baseline for
    C4/C5) gives the reference's ranks, errors and iterations bit for bit."""
    n, pairs = oracle.rmat(14, 16, 0.57, 0.19, 0.19, 2108)
    g = oracle.build_csr(n, pairs)
    h = ref.build_csr_handle(n, pairs)
    v = oracle.csr_view(n, g.in_offsets, g.in_neighbors, g.out_degree)
    try:
        for a, norm in ((0.85, "l1"), (0.95, "l2"), (1.0, "linf")):
            want = ref.pagerank(h, a, 1e-9, norm, 500, trace=True)
            for threads in (1, 3, 8):
                got = oracle.pagerank_mt(v, a, 1e-9, norm, 500, threads=threads, trace=True)
                assert got["iterations"] == want["iterations"]
                assert np.array_equal(got["ranks"], want["ranks"])
                assert np.array_equal(got["err_trace"], want["err_trace"])
    finally:
        ref.free_csr(h)


def test_inplace_rmat_csr_matches_build_csr(oracle, ref):
    """csr_inplace.hpp (the reference arm's C5 builder) gives build_csr's arrays."""
    n, pairs = oracle.rmat(15, 16, 0.57, 0.19, 0.19, 2108)
    want = ref.build_csr(n, pairs)
    h = ref.csr_rmat(15, 16, 0.57, 0.19, 0.19, 2108)
    try:
        got = ref.csr_arrays(h)
    finally:
        ref.free_csr(h)
    for k in ("in_offsets", "in_neighbors", "out_degree", "dangling"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
