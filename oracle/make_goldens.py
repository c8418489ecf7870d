#!/usr/bin/env python3
"""Writes tests/golden/* from the REFERENCE ITSELF (oracle/_ref/libprref.so).

Run here, where /root/reference exists:  python oracle/make_goldens.py small c1 c2 c3

Every golden number below comes from the reference's own build_csr / pagerank /
error_norm / graph generators (compiled from /root/reference by oracle/Makefile);
the oracle restatement and the GPU path are both checked against these files.

  small  fixtures (tests/fixtures/*.mtx, parsed here), the acceptance.cpp:104-132
         oracle-equivalence trial set (seed 4242, 220 trials), known answers
         (test_pagerank.cpp), regular ring (acceptance.cpp:248-259), the
         scale_free_web(2021, 10000, 4, .08) damping/sensitivity cases
         (acceptance.cpp:261-329)
  c1     BASELINE.json configs[0]: RMAT-16, alpha .85, tau 1e-6, L1 (+ other norms)
  c2     configs[1]: RMAT-22 damping sweep, 11 alphas, tau 1e-6, L1
  c3     configs[2]: grid 4096^2, alpha .85, tau 1e-1..1e-10 x {L1,L2,Linf}
  c4     configs[3]: RMAT-26, alpha .85, tau 1e-10, Linf (long: ~30 min, ~20 GB)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from pyoracle import Oracle, Ref  # noqa: E402

GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")
FIXTURE_DIR = "/root/reference/proj/tests/fixtures"
SEED = 2108  # generator seed for every synthetic benchmark graph
NORMS = ["l1", "l2", "linf"]


def parse_mtx(path):
    """Minimal MatrixMarket coordinate parse (graph.hpp:111-199 semantics)."""
    with open(path) as f:
        lines = f.read().splitlines()
    banner = lines[0].split()
    symmetric = banner[4].lower() == "symmetric"
    i = 1
    while lines[i].strip() == "" or lines[i].lstrip().startswith("%"):
        i += 1
    rows, cols, entries = map(int, lines[i].split())
    n = max(rows, cols)
    pairs = []
    seen = 0
    i += 1
    while seen < entries:
        s = lines[i].strip()
        i += 1
        if not s or s.startswith("%"):
            continue
        f = s.split()
        src, dst = int(f[0]) - 1, int(f[1]) - 1
        pairs += [src, dst]
        if symmetric and src != dst:
            pairs += [dst, src]
        seen += 1
    return n, np.array(pairs, np.uint32)


def csr_dict(g):
    return dict(in_offsets=g.in_offsets.tolist(), in_neighbors=g.in_neighbors.tolist(),
                out_degree=g.out_degree.tolist(), dangling=g.dangling.tolist())


def run_dict(R, h, alpha, tol, norm, max_iter=500):
    r = R.pagerank(h, alpha, tol, norm, max_iter, trace=True)
    return dict(alpha=alpha, tol=tol, norm=norm, max_iter=max_iter,
                iterations=r["iterations"], converged=r["converged"],
                ranks=r["ranks"].tolist(), err_trace=r["err_trace"].tolist())


def small(R: Ref):
    out = {"fixtures": {}, "trials": [], "known": {}}
    # --- fixtures -------------------------------------------------------------
    for name in sorted(os.listdir(FIXTURE_DIR)):
        n, pairs = parse_mtx(os.path.join(FIXTURE_DIR, name))
        h = R.build_csr_handle(n, pairs)
        runs = []
        for norm in NORMS:
            for alpha in (0.0, 0.5, 0.85, 1.0):
                for tol in (1e-6, 1e-10):
                    runs.append(run_dict(R, h, alpha, tol, norm))
        runs.append(run_dict(R, h, 1.0, 1e-15, "l1", max_iter=50))  # cap honesty
        runs.append(run_dict(R, h, 0.85, 1e-12, "l1", max_iter=2))
        out["fixtures"][name[:-4]] = dict(n=n, pairs=pairs.tolist(),
                                          csr=csr_dict(R.csr_arrays(h)), runs=runs)
        R.free_csr(h)

    # --- acceptance.cpp:104-132 trial set (statement order is well defined) ---
    rng = R.rng(4242)
    for trial in range(220):
        n = 2 + R.rng_next(rng) % 49
        p = 0.1 + 0.4 * (R.rng_next(rng) % 1000) / 1000.0
        force = trial % 2 == 0
        n_, pairs = R.random_digraph(rng, n, p, force)
        alpha = 0.5 + 0.45 * (R.rng_next(rng) % 1000) / 1000.0
        tol = 1e-8 if trial % 3 == 0 else 1e-6
        norm = NORMS[trial % 3]
        h = R.build_csr_handle(n, pairs)
        got = R.pagerank(h, alpha, tol, norm, 500, trace=True)
        dense = R.dense_pagerank(n, pairs, alpha, tol, norm)
        R.free_csr(h)
        out["trials"].append(dict(n=n, pairs=pairs.tolist(), alpha=alpha, tol=tol, norm=norm,
                                  iterations=got["iterations"], converged=got["converged"],
                                  ranks=got["ranks"].tolist(),
                                  err_trace=got["err_trace"].tolist(),
                                  dense_iterations=dense["iterations"],
                                  dense_ranks=dense["ranks"].tolist()))
    R.rng_free(rng)

    # --- known answers ----------------------------------------------------------
    k = out["known"]
    k["estimates"] = [[a, t, R.estimate_iterations(a, t)]
                      for a, t in [(0.85, 1e-6), (0.95, 1e-6), (0.75, 1e-6), (0.85, 1e-9),
                                   (0.85, 1e-3), (0.5, 0.99)]]
    n, pairs = R.regular_ring(1000, 3)
    h = R.build_csr_handle(n, pairs)
    k["ring_1000_3"] = [[norm, tol, R.pagerank(h, 0.85, tol, norm)["iterations"]]
                        for norm in NORMS for tol in (1e0, 1e-6, 1e-10)]
    R.free_csr(h)
    rng = R.rng(2021)
    n, pairs = R.scale_free_web(rng, 10000, 4, 0.08)
    R.rng_free(rng)
    k["scale_free_10k"] = dict(n=n, m=int(pairs.size // 2), hash_pairs=None)
    h = R.build_csr_handle(n, pairs)
    k["scale_free_10k"]["damping"] = {str(a): R.pagerank(h, a, 1e-6, "l1")["iterations"]
                                      for a in (0.75, 0.85, 0.95)}
    grid = [1e0, 5e-1, 1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4, 1e-4, 5e-5, 1e-5, 5e-6, 1e-6,
            5e-7, 1e-7, 5e-8, 1e-8, 5e-9, 1e-9, 5e-10, 1e-10, 5e-11, 1e-11, 5e-12, 1e-12,
            5e-13, 1e-13, 5e-14, 1e-14, 5e-15, 1e-15, 5e-16, 1e-16]
    sens = []
    for norm in NORMS:
        tr = R.pagerank(h, 0.95, 1e-300, norm, 500, trace=True, want_ranks=False)["err_trace"]
        sens.append(dict(norm=norm, err_trace=tr.tolist()))
    k["scale_free_10k"]["sensitivity_alpha095"] = dict(grid=grid, traces=sens)
    r85 = R.pagerank(h, 0.85, 1e-6, "l1")
    k["scale_free_10k"]["ranks_085"] = r85["ranks"].tolist()
    k["scale_free_10k"]["iterations_085"] = r85["iterations"]
    R.free_csr(h)
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, "small.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("small.json written")


def fingerprint(O: Oracle, g):
    return dict(n=g.vertex_count, e=g.edge_count(), ndangling=int(g.dangling.size),
                h_offsets=O.hash64(g.in_offsets), h_neighbors=O.hash64(g.in_neighbors),
                h_degree=O.hash64(g.out_degree), h_dangling=O.hash64(g.dangling),
                max_in_degree=int(np.diff(g.in_offsets.astype(np.int64)).max()))


def sample_idx(n, k=16384):
    rs = np.random.default_rng(20210806)
    return np.sort(rs.choice(n, size=min(k, n), replace=False)).astype(np.int64)


def rank_summary(ranks, idx):
    top = np.argsort(-ranks, kind="stable")[:1024]
    return dict(sample=ranks[idx], top_idx=top.astype(np.int64), top=ranks[top],
                total=np.sum(ranks.astype(np.longdouble)).astype(np.float64))


def rmat_graph(O, R, scale):
    t = time.time()
    n, pairs = O.rmat(scale, 16, 0.57, 0.19, 0.19, SEED)
    h = R.build_csr_handle(n, pairs)
    g = R.csr_arrays(h)
    fp = fingerprint(O, g)
    fp["raw_edges"] = int(pairs.size // 2)
    fp["h_pairs"] = O.hash64(pairs)
    print(f"rmat{scale}: n={n} e={fp['e']} build {time.time() - t:.1f}s", flush=True)
    return h, g, fp


def c1(O, R):
    h, g, fp = rmat_graph(O, R, 16)
    arrays = {}
    runs = {}
    for norm in NORMS:
        r = R.pagerank(h, 0.85, 1e-6, norm, 500, trace=True)
        runs[norm] = dict(iterations=r["iterations"], converged=r["converged"])
        arrays[f"ranks_{norm}"] = r["ranks"]
        arrays[f"trace_{norm}"] = r["err_trace"]
    R.free_csr(h)
    np.savez_compressed(os.path.join(GOLD, "c1_rmat16.npz"), **arrays)
    with open(os.path.join(GOLD, "c1_rmat16.json"), "w") as f:
        json.dump(dict(config="rmat16 alpha .85 tau 1e-6", seed=SEED, graph=fp, runs=runs),
                  f, indent=1)
    print("c1 written")


def c2(O, R):
    h, g, fp = rmat_graph(O, R, 22)
    idx = sample_idx(g.vertex_count)
    alphas = [0.50, 0.55, 0.60, 0.65, 0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.00]
    t = time.time()
    ref = R.pagerank(h, 0.85, 1e-6, "l1", 500)["ranks"]  # reference_ranks, pagerank.hpp:130
    arrays = dict(sample_idx=idx)
    lanes = []
    for k, a in enumerate(alphas):
        r = R.pagerank(h, a, 1e-6, "l1", 500, trace=True)
        s = rank_summary(r["ranks"], idx)
        for key, v in s.items():
            arrays[f"lane{k}_{key}"] = np.asarray(v)
        arrays[f"lane{k}_trace"] = r["err_trace"]
        lanes.append(dict(alpha=a, iterations=r["iterations"], converged=r["converged"],
                          err_vs_ref=R.error_norm("l1", r["ranks"], ref),
                          loop_ms=r["elapsed_ms"]))
        print(f"  alpha {a}: {r['iterations']} it, {r['elapsed_ms']:.0f} ms", flush=True)
    R.free_csr(h)
    np.savez_compressed(os.path.join(GOLD, "c2_rmat22.npz"), **arrays)
    with open(os.path.join(GOLD, "c2_rmat22.json"), "w") as f:
        json.dump(dict(config="rmat22 damping sweep tau 1e-6 L1", seed=SEED, graph=fp,
                       lanes=lanes, wall_s=time.time() - t), f, indent=1)
    print("c2 written")


def c3(O, R):
    t = time.time()
    n, pairs = O.grid(4096, 0.6, 0.01, SEED)
    h = R.build_csr_handle(n, pairs)
    g = R.csr_arrays(h)
    fp = fingerprint(O, g)
    fp["raw_edges"] = int(pairs.size // 2)
    fp["h_pairs"] = O.hash64(pairs)
    print(f"grid: n={n} e={fp['e']} build {time.time() - t:.1f}s", flush=True)
    idx = sample_idx(n)
    ref = R.pagerank(h, 0.85, 1e-6, "l1", 500)["ranks"]
    taus = [10.0 ** -k for k in range(1, 11)]
    arrays = dict(sample_idx=idx)
    traces = {}
    for norm in NORMS:
        r = R.pagerank(h, 0.85, 1e-10, norm, 500, trace=True)
        traces[norm] = dict(iterations=r["iterations"], converged=r["converged"])
        arrays[f"trace_{norm}"] = r["err_trace"]
        s = rank_summary(r["ranks"], idx)
        for key, v in s.items():
            arrays[f"{norm}_final_{key}"] = np.asarray(v)
        print(f"  {norm}: {r['iterations']} it {r['elapsed_ms']:.0f} ms", flush=True)
    # err_vs_ref per cell: the run capped at the cell's stop iteration gives r_t
    cells = []
    for norm in NORMS:
        tr = arrays[f"trace_{norm}"]
        for tau in taus:
            below = np.nonzero(tr < tau)[0]
            it = int(below[0]) + 1 if below.size else 500
            r = R.pagerank(h, 0.85, tau, norm, 500)
            assert r["iterations"] == it
            cells.append(dict(norm=norm, tol=tau, iterations=it, converged=r["converged"],
                              err_vs_ref=R.error_norm("l1", r["ranks"], ref)))
    R.free_csr(h)
    np.savez_compressed(os.path.join(GOLD, "c3_grid4096.npz"), **arrays)
    with open(os.path.join(GOLD, "c3_grid4096.json"), "w") as f:
        json.dump(dict(config="grid 4096^2 p .6 +1% long-range, alpha .85", seed=SEED, graph=fp,
                       runs=traces, cells=cells, wall_s=time.time() - t), f, indent=1)
    print("c3 written")


def c4(O, R):
    h, g, fp = rmat_graph(O, R, 26)
    del g
    idx = sample_idx(fp["n"])
    r = R.pagerank(h, 0.85, 1e-10, "linf", 500, trace=True)
    arrays = dict(sample_idx=idx, trace=r["err_trace"])
    for key, v in rank_summary(r["ranks"], idx).items():
        arrays[key] = np.asarray(v)
    R.free_csr(h)
    np.savez_compressed(os.path.join(GOLD, "c4_rmat26.npz"), **arrays)
    with open(os.path.join(GOLD, "c4_rmat26.json"), "w") as f:
        json.dump(dict(config="rmat26 alpha .85 tau 1e-10 Linf", seed=SEED, graph=fp,
                       iterations=r["iterations"], converged=r["converged"],
                       loop_ms=r["elapsed_ms"]), f, indent=1)
    print("c4 written")


if __name__ == "__main__":
    O, R = Oracle(), Ref()
    os.makedirs(GOLD, exist_ok=True)
    for what in sys.argv[1:] or ["small", "c1"]:
        {"small": lambda: small(R), "c1": lambda: c1(O, R), "c2": lambda: c2(O, R),
         "c3": lambda: c3(O, R), "c4": lambda: c4(O, R)}[what]()
