timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -8
for c in fib18 ackermann36 reverse16k fibbatch1 fibbatch; do timeout 120 python tools/run_config.py $c --reps 2 2>&1 | tail -2 | head -1; done
timeout 120 python tools/run_config.py fibbatch --reps 2 --variant 2 --trace-out gpurun_out/trace_fibbatch_s4v2.npy 2>&1 | tail -2 | head -1
timeout 120 python tools/run_config.py sortbatch --reps 2 2>&1 | tail -2 | head -1
timeout 120 python tools/run_config.py sortbatch --reps 2 --variant 2 2>&1 | tail -2 | head -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -c 1 -o gpurun_out/prof_ack34_1cta python tools/run_config.py ackermann:3:4 --reps 1 --max-blocks 1 > gpurun_out/ncu_s4b.log 2>&1; tail -1 gpurun_out/ncu_s4b.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 1 -c 1 -o gpurun_out/prof_fibbatch_steady python tools/run_config.py fibbatch --reps 2 > gpurun_out/ncu_s4a.log 2>&1; tail -1 gpurun_out/ncu_s4a.log
