#!/bin/bash
# ncu --set full captures (source-level) of one steady-state step-loop launch per workload
cd "${GRAFT_REPO_ROOT:-.}"
for c in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 1 -c 1 \
      -o gpurun_out/ncu_$c python tools/profile_target.py $c > gpurun_out/ncu_$c.log 2>&1
  tail -2 gpurun_out/ncu_$c.log
done
timeout 300 python tools/probe_overhead.py 2>&1 | tail -6
