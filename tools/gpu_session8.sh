timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/probe_overhead.py 2>&1 | tail -6 | head -2
for c in fib18 ackermann36 reverse16k fibbatch1 fibbatch sortbatch transform22 buildsum22; do timeout 120 python tools/run_config.py $c --reps 2 2>&1 | tail -2 | head -1; done
for c in fibbatch sortbatch; do timeout 120 python tools/run_config.py $c --reps 2 --variant 2 2>&1 | tail -2 | head -1; done
timeout 120 python tools/run_config.py fibbatch --reps 2 --trace-out gpurun_out/trace_fibbatch_s8.npy 2>&1 | tail -1
