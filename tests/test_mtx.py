"""CPU: the library's parallel MatrixMarket parser (prgpu_mtx_parse /
prgpu_mtx_load) against the reference's own
parse_matrix_market / load_matrix_market (oracle/_ref, graph.hpp:111-199,
238-247): identical edge lists in identical order, identical error lines and
messages, for every thread count (ranges split mid-file)."""
import ctypes as C
import os
import random

import numpy as np
import pytest

from conftest import ROOT

THREADS = [1, 2, 3, 5, 8, 17]


@pytest.fixture(scope="module")
def native():
    from paper_2108_02997_b200 import _lib
    return _lib


def parse_native(_lib, text: bytes, threads: int):
    L = _lib.lib()
    n, m, line = C.c_uint32(), C.c_uint64(), C.c_uint64()
    pairs = C.POINTER(C.c_uint32)()
    st = L.prgpu_mtx_parse(text, len(text), threads, C.byref(n), C.byref(pairs), C.byref(m), C.byref(line))
    if st != 0:
        return ("error", st, int(line.value), L.prgpu_last_error().decode())
    arr = np.ctypeslib.as_array(pairs, shape=(2 * m.value,)).copy() if m.value else np.zeros(0, np.uint32)
    L.prgpu_pairs_free(pairs)
    return int(n.value), arr.reshape(-1, 2)


def parse_ref(ref, text: bytes):
    try:
        return ref.parse_mtx(text)
    except ValueError as e:
        line, what = e.args[0]
        return ("error", 5, line, what)


def same(a, b):
    if a[0] == "error" or b[0] == "error":
        return a == b
    return a[0] == b[0] and np.array_equal(a[1], b[1])


# the reference's own cases (test_graph.cpp:33-104)
CASES = [
    "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n2 3\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n2 1\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 2\n1 1\n2 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.5\n",
    "%%MatrixMarket matrix coordinate pattern general\n% comment\n\n2 5 1\n% another\n1 4\n",
    "%%MatrixMarket matrix coordinate pattern\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1 0\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "%%MatrixMarket matrix coordinate pattern skew-symmetric\n1 1 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 x\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n% c\n2 2 1\n3 1\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n",
    "%%MatrixMarket matrix coordinate pattern general\n0 0 0\n",
    # more edges of the language
    "",
    "%%MatrixMarket matrix coordinate pattern general",
    "%%MatrixMarket matrix coordinate pattern general\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2",
    "%%MatrixMarket matrix coordinate pattern general\r\n3 3 2\r\n1 2\r\n\t2 3 \r\n",
    "%%MATRIXMARKET MATRIX Coordinate Pattern General\n3 3 1\n1 2\n",
    "%%MatrixMarket MATRIX Coordinate Pattern General\n3 3 1\n1 2\n",
    "%%MatrixMarket matrix coordinate integer general\n3 3 2\n1 2 -7\n2 3 1e400\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 nan\n2 3 inf\n3 1 +1\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 0x10\n2 3 .5\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\nthis line is never read\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n+1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2 3\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n4294967296 1 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n4294967295 1 1\n4294967295 1\n",
    "%%MatrixMarket matrix coordinate pattern general extra\n1 1 0\n",
    "  %%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
]


def test_reference_cases_every_thread_count(native, ref):
    for text in CASES:
        want = parse_ref(ref, text.encode())
        for t in THREADS:
            got = parse_native(native, text.encode(), t)
            assert same(got, want), (text, t, got, want)


def random_mtx(rng: random.Random):
    sym = rng.random() < 0.3
    field = rng.choice(["pattern", "real", "integer"])
    rows, cols = rng.randint(1, 40), rng.randint(1, 40)
    entries = rng.randint(0, 120)
    out = [f"%%MatrixMarket matrix coordinate {field} {'symmetric' if sym else 'general'}"]
    if rng.random() < 0.3:
        out.append("% size follows")
    out.append(f"{rows} {cols} {entries}")
    nl = entries + rng.randint(-3, 6)
    bad = rng.random() < 0.4
    for i in range(max(nl, 0)):
        r = rng.random()
        if r < 0.05:
            out.append("")
        elif r < 0.1:
            out.append("% comment " + str(i))
        else:
            a, b = rng.randint(1, rows), rng.randint(1, cols)
            sep = rng.choice([" ", "\t", "  "])
            line = f"{a}{sep}{b}"
            if field != "pattern":
                line += sep + rng.choice(["1", "-2.5", "3e7", "0.125", "inf", "7"])
            if bad and rng.random() < 0.03:
                line = rng.choice([f"{a}", f"{a} x", f"{rows + 1} {b}", f"{a} {b} {b} {b}", "1.0 2"])
            if rng.random() < 0.1:
                line += "\r"
            out.append(line)
    text = "\n".join(out) + ("\n" if rng.random() < 0.8 else "")
    return text.encode()


def test_random_files_match_reference(native, ref):
    rng = random.Random(2108)
    for trial in range(400):
        text = random_mtx(rng)
        want = parse_ref(ref, text)
        for t in (1, 3, 7):
            got = parse_native(native, text, t)
            assert same(got, want), (trial, t, text[:300], got, want)


def test_file_load_and_large_input(native, ref, oracle, tmp_path):
    """load_matrix_market on a generated RMAT-16 file (1M lines): the same
    edge list as the reference's; file errors name the file."""
    n, pairs = oracle.rmat(16, 16, 0.57, 0.19, 0.19, 5)
    p = pairs.reshape(-1, 2).astype(np.int64) + 1
    path = tmp_path / "rmat16.mtx"
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate pattern general\n% generated\n")
        f.write(f"{n} {n} {len(p)}\n")
        np.savetxt(f, p, fmt="%d")
    import paper_2108_02997_b200 as prl
    el = prl.load_matrix_market(path)
    rn, rp = ref.load_mtx(str(path))
    assert el.vertex_count == rn == n
    assert np.array_equal(el.edges, rp)
    assert np.array_equal(el.edges, pairs.reshape(-1, 2))
    with pytest.raises(RuntimeError, match="cannot open graph file: .*missing.mtx"):
        prl.load_matrix_market(tmp_path / "missing.mtx")
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n")
    with pytest.raises(RuntimeError) as ei:
        prl.load_matrix_market(bad)
    with pytest.raises(RuntimeError) as er:
        ref.load_mtx(str(bad))
    assert str(ei.value) == str(er.value) == f"{bad}: line 3: entry (3, 1) out of range for 2 x 2"


def test_parse_matrix_market_api(native):
    import paper_2108_02997_b200 as prl
    el = prl.parse_matrix_market("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n2 1\n")
    assert el.vertex_count == 2 and el.edges.tolist() == [[1, 0], [0, 1]]
    with pytest.raises(prl.MtxParseError) as e:
        prl.parse_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n")
    assert e.value.line() == 4 and str(e.value) == "line 4: unexpected end of file: got 1 of 2 entries"
