#!/bin/bash
# source-level ncu of the step loop (both builds) on one 5F shard and fib(18); the reports come back
# in gpurun_out/ for `ncu -i ... --page source --csv` here
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for c in ${@:-fibbatch1 fib18}; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:step_loop -c 4 \
      -o gpurun_out/src_$c python tools/profile_target.py $c > gpurun_out/src_$c.log 2>&1; echo "ncu $c rc=$?"
done
ls -la gpurun_out
