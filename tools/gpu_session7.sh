timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/probe_overhead.py 2>&1 | tail -8
