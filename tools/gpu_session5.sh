timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 120 python tools/run_config.py ackermann:3:4 --reps 1 --max-blocks 1 --profile 2>&1 | tail -2
timeout 120 python tools/run_config.py ackermann:3:4 --reps 1 --profile 2>&1 | tail -2
timeout 120 python tools/run_config.py fib18 --reps 1 --profile 2>&1 | tail -2
timeout 120 python tools/run_config.py mergesort:1024:1 --reps 1 --profile 2>&1 | tail -2
timeout 120 python tools/run_config.py fibbatch --reps 2 --profile 2>&1 | tail -3
timeout 120 python tools/run_config.py fibbatch --reps 2 --profile --variant 2 2>&1 | tail -3
