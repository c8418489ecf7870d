PYTHONPATH=. PRGPU_TIMING_LOG=1 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -12
PYTHONPATH=. timeout 300 python scripts/e2e_probe.py 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 3
