"""CPU: the C-ABI library loads, exports every symbol include/prgpu.h declares,
and fails loudly (no CPU fallback) when no GPU is visible."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "prgpu.h")
LIB = os.path.join(ROOT, "paper_2108_02997_b200", "libprgpu.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"PRGPU_API\s+[\w\s\*]+?\b(prgpu_\w+)\s*\(", text)))


def test_header_declares_the_api():
    syms = declared_symbols()
    assert "prgpu_pagerank" in syms and "prgpu_graph_build" in syms
    from paper_2108_02997_b200 import _lib
    assert sorted(_lib.EXPORTS) == syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libprgpu.so not built (run __graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (prgpu_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_loads_and_reports_version():
    from paper_2108_02997_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.prgpu_version()


def test_no_cpu_fallback_without_gpu():
    """With no CUDA device the engine refuses (RuntimeError), never computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import numpy as np
    import paper_2108_02997_b200 as prl
    with pytest.raises(RuntimeError, match="no CUDA device"):
        prl.build_csr(prl.EdgeList(2, np.array([[0, 1], [1, 0]], np.uint32)))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        prl.error_norm(prl.NormKind.L1, [0.5, 0.5], [0.5, 0.5])
