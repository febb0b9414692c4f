#!/bin/bash
# phase cycle accounting (profiling build) of the narrow sweeps: where a chain step's cycles go
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/${PH_OUT:-phases}.log
: > $out
timeout 300 python tools/run_config.py fibbatch1 --profile 3000 --reps 2 >> $out 2>&1; echo "rc=$?" >> $out
timeout 300 python tools/run_config.py fibbatch --profile 50000 --reps 2 >> $out 2>&1; echo "rc=$?" >> $out
timeout 300 python tools/run_config.py fib18 --profile --reps 2 >> $out 2>&1; echo "rc=$?" >> $out
cat $out
