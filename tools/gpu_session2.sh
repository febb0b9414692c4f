set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5
for c in fib18 ackermann36 reverse16k fibbatch1 fibbatch; do timeout 120 python tools/run_config.py $c --reps 2 2>&1 | tail -3; done
timeout 300 python tools/run_config.py mergesort16k --reps 1 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err; tail -3 gpurun_out/bench_s2.err; cat gpurun_out/bench_s2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s2.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1; tail -5 gpurun_out/launches_s2.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -c 1 -o gpurun_out/prof_fibbatch python tools/run_config.py fibbatch --reps 1 > gpurun_out/ncu_s2.log 2>&1; tail -3 gpurun_out/ncu_s2.log
