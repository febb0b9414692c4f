#!/bin/bash
# quick iteration: GPU parity suite + timelines of the batched/wide configs + latency configs
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -x -q -m gpu --timeout 240 --timeout_method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-1}; do for c in fibbatch sortbatch buildsum22 transform22; do timeout 300 python tools/sweep_timeline.py $c --variant $v | python -c "
import json,sys; d=json.load(sys.stdin); print('v$v', d['name'], round(d['kernel_ms'],2), [(b['active'], b['ms'], b['us_per_sweep']) for b in d['buckets']])"; done; done 2>&1
for c in ackermann36 fib18 reverse16k; do timeout 300 python tools/run_config.py $c --reps 2 2>&1 | tail -2 | head -1 | cut -c1-200; done
