#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/ra_compare.py fib18 ackermann36 reverse16k transform22 buildsum22 fibbatch_s1 sortbatch_s1 fibbatch sortbatch mergesort16k > gpurun_out/ra.log 2>&1
TRS_B200_PROFILE_BUILD=1 timeout 300 python tools/run_config.py fib18 --profile --reps 2 > gpurun_out/prof_fib18.log 2>&1
TRS_B200_PROFILE_BUILD=1 timeout 300 python tools/run_config.py transform22 --profile --reps 2 > gpurun_out/prof_t22.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-configs > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 2400 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
