"""Helpers for the CLI and acceptance tests: the reference's fixture graphs
written back as MatrixMarket files from tests/golden/small.json (which holds
their edge lists as the reference's parser read them), and a runner for
tools/pagerank-lab."""
import json
import os
import subprocess

from conftest import GOLD, ROOT

CLI = os.path.join(ROOT, "tools", "pagerank-lab")
ACCEPTANCE = os.path.join(ROOT, "tests", "cpp", "build", "acceptance")
# tools/Makefile compiles this path into the acceptance binary
FIXTURE_DIR = "/root/repo/tests/cpp/build/fixtures"


def write_fixtures(where: str) -> None:
    """<where>/<name>.mtx for every fixture of small.json (general, 1-based)."""
    os.makedirs(where, exist_ok=True)
    with open(os.path.join(GOLD, "small.json")) as f:
        fx = json.load(f)["fixtures"]
    for name, g in fx.items():
        pairs = g["pairs"]
        m = len(pairs) // 2
        lines = ["%%MatrixMarket matrix coordinate pattern general", f"{g['n']} {g['n']} {m}"]
        lines += [f"{pairs[2 * i] + 1} {pairs[2 * i + 1] + 1}" for i in range(m)]
        path = os.path.join(where, name + ".mtx")
        with open(path + ".tmp", "w") as out:
            out.write("\n".join(lines) + "\n")
        os.replace(path + ".tmp", path)


def cli(*args, stderr=False, timeout=600):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, (r.stdout + r.stderr) if stderr else r.stdout


def body_rows(path) -> int:
    with open(path) as f:
        return sum(1 for i, line in enumerate(f) if i > 0 and line.strip())
