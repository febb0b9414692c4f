#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export TRS_B200_JIT_VERBOSE=1
timeout 900 python tools/ra_compare.py fib18 ackermann36 reverse16k transform22 buildsum22 fibbatch_s1 sortbatch_s1 fibbatch sortbatch mergesort16k > gpurun_out/ra.log 2>&1
unset TRS_B200_JIT_VERBOSE
timeout 2700 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
