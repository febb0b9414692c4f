#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/ra_compare.py transform22 fib18 ackermann36 buildsum22 fibbatch sortbatch mergesort16k > gpurun_out/ra.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
