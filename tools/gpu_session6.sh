timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6
for c in fib18 ackermann36 reverse16k fibbatch1 fibbatch sortbatch transform22 buildsum22; do timeout 120 python tools/run_config.py $c --reps 2 2>&1 | tail -2 | head -1; done
timeout 120 python tools/run_config.py ackermann:3:4 --reps 1 --profile 2>&1 | tail -1
timeout 120 python tools/run_config.py ackermann:3:4 --reps 1 --profile --small-enter 0 2>&1 | tail -1
timeout 120 python tools/run_config.py fibbatch --reps 2 --profile 2>&1 | tail -1
timeout 120 python tools/run_config.py fibbatch --reps 2 --variant 2 --trace-out gpurun_out/trace_fibbatch_s6v2.npy 2>&1 | tail -2 | head -1
timeout 120 python tools/run_config.py fibbatch --reps 2 --trace-out gpurun_out/trace_fibbatch_s6v1.npy 2>&1 | tail -2 | head -1
timeout 300 python tools/run_config.py mergesort16k --reps 1 2>&1 | tail -2 | head -1
