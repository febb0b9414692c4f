#!/bin/bash
# compute-sanitizer over the engine's kernels (tools/sanitize_cases.py):
# memcheck, racecheck, synccheck and initcheck, each under a timeout.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  case $tool in
    memcheck) modes=default,sync,grid,interp,gc1,validate2; n=10 ;;
    *) modes=default,sync,grid,gc1; n=4 ;;
  esac
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py $modes $n > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log
done
