set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30
for c in fib18 ackermann36 transform22 buildsum22 reverse16k; do timeout 120 python tools/run_config.py $c --ref --reps 2 2>&1 | tail -4; done
timeout 120 python tools/run_config.py fibbatch1 --reps 2 2>&1 | tail -3
timeout 300 python tools/run_config.py mergesort16k --reps 1 2>&1 | tail -3
