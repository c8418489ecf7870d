"""CPU: host-side logic of the Python mirror (no GPU calls) — MatrixMarket
parsing (graph.hpp:111-199 / test_graph.cpp:82-104), CSV number formatting
(csv.hpp:17-21, checked against std::to_chars), the estimator, grids,
fused-sweep cell extraction and detect_sensitivity (sweep.hpp:262-310)."""
import math
import os
import subprocess

import numpy as np
import pytest

import paper_2108_02997_b200 as prl
from paper_2108_02997_b200.pagerank_lab import _cells_from_trace


def parse(text):
    return prl.parse_matrix_market(text)


def test_parse_pattern_symmetric_weights():
    el = parse("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n2 3\n")
    assert el.vertex_count == 3 and el.edges.tolist() == [[0, 1], [1, 2]]
    el = parse("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n2 1\n")
    assert el.edges.tolist() == [[1, 0], [0, 1]]
    el = parse("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 2\n1 1\n2 1\n")
    assert len(el.edges) == 3
    el = parse("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.5\n")
    assert el.edges.tolist() == [[0, 1]]
    el = parse("%%MatrixMarket matrix coordinate pattern general\n% c\n\n2 5 1\n% x\n1 4\n")
    assert el.vertex_count == 5


@pytest.mark.parametrize("text,line", [
    ("%%MatrixMarket matrix coordinate pattern\n1 1 0\n", 1),
    ("%%MatrixMarket matrix array real general\n1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate pattern skew-symmetric\n1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 x\n", 2),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2\n", 2),
    ("%%MatrixMarket matrix coordinate pattern general\n% c\n2 2 1\n3 1\n", 4),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n", 3),
    ("%%MatrixMarket matrix coordinate pattern general\n0 0 0\n", 2),
])
def test_parse_errors_name_the_line(text, line):
    with pytest.raises(prl.MtxParseError) as ei:
        parse(text)
    assert ei.value.line() == line


def test_load_matrix_market_names_the_file():
    with pytest.raises(RuntimeError, match="cannot open graph file: no_such_file.mtx"):
        prl.load_matrix_market("no_such_file.mtx")


def test_format_double_matches_std_to_chars(tmp_path):
    """csv.hpp:17-21 uses std::to_chars; the Python mirror must print the same."""
    src = tmp_path / "tc.cpp"
    src.write_text('#include <charconv>\n#include <cstdio>\n#include <cstdlib>\n'
                   'int main(int c, char** v){ for(int i=1;i<c;++i){ double x=std::strtod(v[i],nullptr);'
                   ' char b[64]; auto r=std::to_chars(b,b+64,x); *r.ptr=0; std::puts(b);} }\n')
    exe = tmp_path / "tc"
    subprocess.run(["g++", "-std=c++20", "-O1", str(src), "-o", str(exe)], check=True)
    rs = np.random.default_rng(5)
    vals = [0.0, 1.0, 100.0, 0.85, 1e-06, 5e-10, 1e-10, 123456789.0, 1e21, 1e22, 0.1, 2.5e-5,
            1234.5678, 1e16, 12345678901234567.0, 0.000123]
    vals += list(rs.random(200)) + list(10.0 ** rs.uniform(-12, 12, 200)) + list(rs.random(50) * 1e3)
    args = [repr(float(v)) for v in vals]
    out = subprocess.run([str(exe)] + args, capture_output=True, text=True, check=True).stdout.split()
    for v, want in zip(vals, out):
        assert prl.format_double(v) == want, (v, want)


def test_estimator_and_grids():
    assert [prl.estimate_iterations(a, t) for a, t in
            [(0.85, 1e-6), (0.95, 1e-6), (0.75, 1e-6), (0.85, 1e-9), (0.85, 1e-3)]] == [85, 269, 48, 128, 43]
    for bad in [(1.0, 1e-6), (0.0, 1e-6), (0.85, 1.0), (0.85, 0.0)]:
        with pytest.raises(ValueError):
            prl.estimate_iterations(*bad)
    assert len(prl.default_damping_grid()) == 11 and len(prl.default_tolerance_grid()) == 21
    assert prl.parse_norm("LInf") == prl.NormKind.LInf and prl.parse_norm("l3") is None


def test_fused_cells_from_trace():
    """A (tau, norm) cell stops at the first iteration whose error is < tau
    (pagerank.hpp:99); if none does, it reports the cap, unconverged."""
    tr = np.zeros((5, 4))
    tr[:, 0] = [1.0, 0.1, 0.01, 1e-3, 1e-4]
    assert _cells_from_trace(tr, 5, prl.NormKind.L1, 0.05, 500) == (3, True)
    assert _cells_from_trace(tr, 5, prl.NormKind.L1, 1e-3, 500) == (5, True)
    assert _cells_from_trace(tr, 5, prl.NormKind.L1, 1e-9, 5) == (5, False)
    assert _cells_from_trace(tr, 5, prl.NormKind.L1, 2.0, 500) == (1, True)


def test_sweep_csv_row_and_sensitivity():
    r = prl.SweepRecord("g,x", 3, 2, 0.85, 1e-06, prl.NormKind.L2, 7, True, 1.5, 0.0)
    assert prl.sweep_csv_row(r) == '"g,x",3,2,0.85,1e-06,l2,7,true,1.5,0'
    grid = [1e-1, 1e-2, 1e-3]
    recs = [prl.SweepRecord("g", 1, 1, 0.95, t, prl.NormKind.L1, it, conv)
            for t, it, conv in zip(grid, [1, 3, 500], [True, True, False])]
    rep = prl.detect_sensitivity(recs)
    assert rep[0].first_failing_tolerance == 1e-3 and rep[0].single_iteration_tolerances == [1e-1]
    with pytest.raises(ValueError):  # the L2 group misses one grid tolerance
        prl.detect_sensitivity(recs + [prl.SweepRecord("g", 1, 1, .95, t, prl.NormKind.L2, 1, True)
                                       for t in grid[:2]])
    with pytest.raises(ValueError):
        prl.SweepPlan(graphs=[]).validate()
    with pytest.raises(ValueError):
        prl.PageRankConfig(alpha=2.0).validate()
