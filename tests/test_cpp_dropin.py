"""The C++ drop-in header: compiles here (CPU) against libprgpu.so, runs on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2108_02997_b200")


def build(out):
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", SRC, "-o", out, "-L", LIBDIR, "-lprgpu",
           f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_dropin_compiles(tmp_path):
    """The header is source-compatible with code written against the reference API."""
    build(str(tmp_path / "test_dropin"))


@pytest.mark.gpu
def test_dropin_runs_on_gpu(tmp_path):
    exe = str(tmp_path / "test_dropin")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "PASS" in r.stdout


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers not present (GPU box)")
def test_dropin_beside_reference_reporting_headers(tmp_path):
    """The drop-in together with the reference's own stats.hpp (mean-ratio
    reporting), csv.hpp and chart.hpp: compiles without name clashes and the
    host-only reporting path runs (north_star: the sweep drivers and
    mean-ratio reporting keep their API)."""
    exe = str(tmp_path / "rep")
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin_reporting.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", "-I", REF_INCLUDE, src, "-o", exe, "-L", LIBDIR,
                    "-lprgpu", f"-Wl,-rpath,{LIBDIR}"], check=True, capture_output=True, text=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
