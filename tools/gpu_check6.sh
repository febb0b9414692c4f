#!/bin/bash
# refcount-free step loop + run-ahead defaults: full GPU suite, A/B, bench
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/rc_ab.py > gpurun_out/rc_ab.log 2>&1; echo "rc_ab rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
