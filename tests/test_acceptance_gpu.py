"""The reference's own acceptance suite (/root/reference/proj/tests/acceptance.cpp),
compiled UNMODIFIED against the B200 drop-in (tools/Makefile: a shadow
include tree maps <pagerank_lab/{graph,norms,pagerank,sweep}.hpp> to
<pagerank_b200/dropin.hpp>; stats/csv/chart and the test support headers are
the reference's), with PAGERANK_LAB_CLI_PATH = tools/pagerank-lab.  All ten
criteria must print PASS on the B200."""
import os
import subprocess

import pytest

from cli_support import ACCEPTANCE, CLI, FIXTURE_DIR, write_fixtures

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(ACCEPTANCE), reason="acceptance binary not built (tools/Makefile)")
def test_reference_acceptance_suite_on_b200():
    assert os.path.exists(CLI)
    write_fixtures(FIXTURE_DIR)
    r = subprocess.run([ACCEPTANCE], capture_output=True, text=True, timeout=900)
    lines = [x for x in r.stdout.splitlines() if x.startswith(("PASS", "FAIL"))]
    assert len(lines) == 10, r.stdout + r.stderr
    assert all(x.startswith("PASS") for x in lines), r.stdout
    assert r.returncode == 0
