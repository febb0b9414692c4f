#!/bin/bash
# resident arena on/off (its shared memory also sets the L1 carve-out) on the latency-bound configs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/resident_ab.log
: > $out
for c in fib18 reverse16k fibbatch1 ackermann36 mergesort16k; do
  for flag in "" "--no-resident"; do
    echo "== $c $flag" >> $out
    timeout 300 python tools/run_config.py $c $flag --reps 3 2>&1 | grep '"rep": 2' >> $out
  done
done
cat $out
