#!/bin/bash
# compute-sanitizer over the engine's kernels (tools/sanitize_cases.py):
# memcheck, racecheck, synccheck and initcheck, each under a timeout.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  # spin-waiting (grid barrier, parked CTAs) is instrumented too: keep the cases small
  case $tool in
    memcheck) modes=default,sync,grid,interp,gc1,gc1u; n=3; k=10 ;;
    racecheck) modes=default,gc1u; n=1; k=4 ;;
    *) modes=default,grid,gc1u; n=2; k=5 ;;
  esac
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py $modes $n $k > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log
done
