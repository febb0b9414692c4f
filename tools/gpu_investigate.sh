#!/bin/bash
# probes + per-sweep timelines + phase-cycle profiles of the latency-bound configs
cd "${GRAFT_REPO_ROOT:-.}"
python - <<'PY' > gpurun_out/probe.log 2>&1
import sys; sys.path.insert(0, '.')
from paper_2009_07174_b200 import api
for b in (4, 8, 16, 32):
    print(b, api.gather_probe(0, 4 << 30, b, 5), flush=True)
PY
cat gpurun_out/probe.log
for c in fibbatch sortbatch buildsum22 transform22; do timeout 300 python tools/sweep_timeline.py $c --save gpurun_out/tl_$c.npy; done > gpurun_out/timeline.log 2>&1
cat gpurun_out/timeline.log
for c in ackermann36 fib18 reverse16k; do timeout 300 python tools/run_config.py $c --reps 2 --profile 2>&1 | tail -3; done > gpurun_out/prof_latency.log 2>&1
cat gpurun_out/prof_latency.log
