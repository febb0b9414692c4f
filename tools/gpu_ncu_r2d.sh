#!/bin/bash
# ncu --set full of the step loop at HEAD for the configs the last changes moved
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/*
for c in fibbatch fibbatch1 fib18 buildsum22; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:step_loop -c 4 \
      -o /tmp/ncu/ncu_$c python tools/profile_target.py $c > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
cp profiles/traffic.json gpurun_out/traffic_before.json
python tools/ncu_summary.py /tmp/ncu r2d gpurun_out > gpurun_out/ncu_summary.log 2>&1; echo "summary rc=$?"
