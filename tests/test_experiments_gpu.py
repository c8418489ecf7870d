"""The tuning build (make -C paper_2108_02997_b200/csrc EXPERIMENTS=1 ->
build_alt/libprgpu_exp.so) keeps the measured-negative switches of
profiles/r2_c5_l2_experiments.md compiled in; its split pull is still a
correct solver: the split parity test runs against it in a subprocess (one
library per process)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

LIB = os.path.join(ROOT, "build_alt", "libprgpu_exp.so")


@pytest.mark.skipif(not os.path.exists(LIB), reason="tuning build not present")
def test_tuning_build_split_pull_parity():
    env = dict(os.environ, PRGPU_LIB=LIB)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-k", "split_pull",
                        os.path.join(ROOT, "tests", "test_parity_gpu.py")], env=env, capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "2 passed" in r.stdout
