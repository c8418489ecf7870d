"""tools/pagerank-lab — the reference CLI's subcommands over the B200 path
(/root/reference/proj/tools/main.cpp).  The cases follow
the reference's own CLI tests (tests/test_cli.cpp): same commands, same
expected rows, cells and exit codes.  Host-only commands (ratios, estimate,
chart on a given CSV, flag errors) run here; the ones that solve PageRank run
on the GPU."""
import os

import pytest

from cli_support import CLI, body_rows, cli, write_fixtures

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="tools/pagerank-lab not built")

HEADER = "graph,vertices,edges,alpha,tolerance,norm,iterations,converged,time_ms,err_vs_ref\n"


def csv_file(tmp_path, name, body):
    p = tmp_path / name
    p.write_text(HEADER + body)
    return p


def test_ratios_hand_computed_cells(tmp_path):
    p = csv_file(tmp_path, "gm.csv", "gmean,1,1,0.85,1e-06,l1,56.91,true,1,0\n"
                                     "gmean,1,1,0.85,1e-06,l2,27.50,true,1,0\n"
                                     "gmean,1,1,0.85,1e-06,linf,10.21,true,1,0\n")
    rc, out = cli("ratios", "--input", p, "--metric", "iterations", "--method", "gm-ratio")
    assert rc == 0
    assert out.splitlines() == ["method,baseline,mean:l1,mean:l2,mean:linf,ratio:l1,ratio:l2,ratio:linf",
                                "gm-ratio,l1,56.91,27.50,10.21,1.00,0.48,0.18"]
    rc, out = cli("ratios", "--input", p, "--metric", "iterations", "--method", "gm-ratio", "--baseline", "linf")
    assert out.splitlines()[1] == "gm-ratio,linf,56.91,27.50,10.21,5.57,2.69,1.00"
    rc, a = cli("ratios", "--input", p, "--method", "all")
    assert rc == 0 and len(a.splitlines()) == 7  # header + six methods
    assert cli("ratios", "--input", p, "--method", "all")[1] == a  # byte-identical


def test_ratios_constant_incomplete_and_warning(tmp_path):
    p = csv_file(tmp_path, "c.csv", "g,1,1,0.85,1e-06,l1,7,true,1,0\ng,1,1,0.85,1e-06,l2,7,true,1,0\n")
    rc, out = cli("ratios", "--input", p, "--method", "ratio-am")
    assert rc == 0 and out.splitlines()[1] == "ratio-am,l1,,,1.00,1.00"
    p = csv_file(tmp_path, "i.csv", "g,1,1,0.85,1e-06,l1,7,true,1,0\ng,1,1,0.85,1e-05,l1,9,true,1,0\n"
                                    "g,1,1,0.85,1e-06,l2,5,true,1,0\n")
    assert cli("ratios", "--input", p)[0] == 1
    p = csv_file(tmp_path, "n.csv", "g,1,1,0.85,1e-06,l1,500,false,1,0\ng,1,1,0.85,1e-06,l2,40,true,1,0\n")
    rc, out = cli("ratios", "--input", p, "--method", "gm-ratio", stderr=True)
    assert "warning: 1 non-converged cell" in out
    assert cli("ratios", "--input", p, "--metric", "edges")[0] == 2
    assert cli("ratios", "--input", p, "--method", "nope")[0] == 2
    assert cli("ratios", "--input", tmp_path / "missing.csv")[0] == 1


def test_estimate():
    for a, t, want in ((0.85, 1e-6, "85"), (0.95, 1e-6, "269"), (0.75, 1e-6, "48"), (0.85, 1e-9, "128"),
                       (0.85, 1e-3, "43")):
        assert cli("estimate", "--alpha", a, "--tolerance", t) == (0, want + "\n")
    assert cli("estimate", "--alpha", 1.2, "--tolerance", 1e-6)[0] == 2
    assert cli("estimate", "--alpha=0.85", "--tolerance=1e-6") == (0, "85\n")


def test_chart_from_csv_and_rejections(tmp_path):
    body = "".join(f"g,1,1,0.85,{t},{nm},{i},true,1,0\n"
                   for nm, base in (("l1", 10), ("l2", 8), ("linf", 6)) for t, i in ((1e-2, base), (1e-4, 2 * base)))
    p = csv_file(tmp_path, "s.csv", body)
    svg = tmp_path / "c.svg"
    rc, _ = cli("chart", "--input", p, "--x", "tolerance", "--y", "iterations", "--series", "norm", "--log-x",
                "--out", svg)
    assert rc == 0 and svg.read_text().count("<polyline") == 3
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n1,2\n")
    assert cli("chart", "--input", bad, "--x", "nope", "--y", "b", "--out", tmp_path / "x.svg")[0] == 2
    empty = tmp_path / "empty.csv"
    empty.write_text("a,b\n")
    assert cli("chart", "--input", empty, "--x", "a", "--y", "b", "--out", tmp_path / "x.svg")[0] == 2


def test_flag_errors_exit_2():
    assert cli("no-such-command")[0] == 2
    assert cli()[0] == 2
    assert cli("run", "--graph", "x.mtx", "--bogus", "1")[0] == 2
    assert cli("run")[0] == 2  # --graph required
    assert cli("sweep-damping", "--graph", "x.mtx")[0] == 2  # --csv required
    assert cli("estimate", "--alpha", "abc", "--tolerance", "1e-6")[0] == 2
    assert cli("--help")[0] == 0 and cli("run", "--help")[0] == 0


# ---- commands that solve PageRank (GPU) ------------------------------------
@pytest.fixture(scope="module")
def fx(tmp_path_factory):
    d = tmp_path_factory.mktemp("fixtures")
    write_fixtures(str(d))
    return lambda name: str(d / name)


@pytest.mark.gpu
def test_run_records_and_exit_codes(fx, tmp_path):
    rc, out = cli("run", "--graph", fx("two_cycle.mtx"), "--alpha", 0.85, "--tolerance", 1e-6, "--norm", "l1",
                  "--repeat", 1)
    f = out.splitlines()[0].split(",")
    assert rc == 0 and len(f) == 10 and f[0] == "two_cycle" and f[1:3] == ["2", "2"] and f[6:8] == ["1", "true"]
    rc, out = cli("run", "--graph", fx("tiny_web.mtx"), "--alpha", 0.85, "--tolerance", 1e-6, "--max-iter", 2,
                  "--repeat", 1)
    assert rc == 3 and out.splitlines()[0].split(",")[7] == "false"
    assert cli("run", "--graph", fx("two_cycle.mtx"), "--alpha", 1.5)[0] == 2
    assert cli("run", "--graph", fx("two_cycle.mtx"), "--norm", "l7")[0] == 2
    assert cli("run", "--graph", tmp_path / "missing.mtx")[0] == 1
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 x\n")
    assert cli("run", "--graph", bad)[0] == 1


@pytest.mark.gpu
def test_sweeps_row_counts_and_grids(fx, tmp_path):
    c = tmp_path / "o.csv"
    assert cli("compare-norms", "--graphs", fx("two_cycle.mtx"), fx("star.mtx"), fx("tiny_web.mtx"),
               "--repeat", 1, "--csv", c)[0] == 0
    assert body_rows(c) == 9
    assert cli("sweep-damping", "--graph", fx("star.mtx"), "--repeat", 1, "--csv", c)[0] == 0
    assert body_rows(c) == 11
    assert cli("sweep-tolerance", "--graph", fx("star.mtx"), "--repeat", 1, "--csv", c)[0] == 0
    assert body_rows(c) == 63
    assert cli("sweep-damping", "--graph", fx("star.mtx"), "--alpha-from", 0.7, "--alpha-to", 0.9,
               "--alpha-step", 0.1, "--repeat", 1, "--csv", c)[0] == 0
    assert body_rows(c) == 3
    assert cli("sweep-damping", "--graph", fx("star.mtx"), "--alpha-from", 0.7, "--repeat", 1, "--csv", c)[0] == 2
    assert cli("sweep-tolerance", "--graph", fx("star.mtx"), "--tol-grid", "1e-2,1e-4", "--norms", "l1,linf",
               "--repeat", 1, "--csv", c)[0] == 0
    assert body_rows(c) == 4


@pytest.mark.gpu
def test_sweep_csv_fused_equals_per_cell_and_charts(fx, tmp_path):
    """The fused sweep (one batched run per graph, cells off the norm trace)
    and --per-cell-timing (every cell run on its own, sweep.hpp:173-192)
    write the same CSV except the time column; the damping sweep is monotone
    and the tolerance sweep charts one polyline per norm."""
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    g = [fx("star.mtx"), fx("tiny_web.mtx")]
    assert cli("sweep-tolerance", "--graphs", *g, "--repeat", 1, "--csv", a)[0] == 0
    assert cli("sweep-tolerance", "--graphs", *g, "--repeat", 1, "--per-cell-timing", "--csv", b)[0] == 0
    ra = [r.split(",") for r in a.read_text().splitlines()]
    rb = [r.split(",") for r in b.read_text().splitlines()]
    assert len(ra) == len(rb) == 1 + 2 * 63
    t = ra[0].index("time_ms")
    assert [r[:t] + r[t + 1:] for r in ra] == [r[:t] + r[t + 1:] for r in rb]
    svg = tmp_path / "c.svg"
    assert cli("chart", "--input", a, "--x", "tolerance", "--y", "iterations", "--series", "norm", "--log-x",
               "--out", svg)[0] == 0
    assert svg.read_text().count("<polyline") == 3
    assert cli("sweep-damping", "--graph", fx("star.mtx"), "--repeat", 1, "--csv", a)[0] == 0
    its = [int(r.split(",")[6]) for r in a.read_text().splitlines()[1:]]
    assert its == sorted(its)
