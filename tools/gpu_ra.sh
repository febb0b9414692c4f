#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python tools/ra_compare.py fib18 ackermann36 reverse16k sortbatch_s1 fibbatch_s1 sortbatch mergesort16k > gpurun_out/ra.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
