timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for v in 1 2; do
for c in fib18 ackermann36 reverse16k fibbatch1; do timeout 120 python tools/run_config.py $c --reps 2 --variant $v 2>&1 | tail -2 | head -1; done
timeout 120 python tools/run_config.py fibbatch --reps 2 --variant $v --trace-out gpurun_out/trace_fibbatch_v$v.npy 2>&1 | tail -2 | head -1
timeout 120 python tools/run_config.py ackermann:3:4 --reps 1 --variant $v --trace-out gpurun_out/trace_ack34_v$v.npy 2>&1 | tail -2 | head -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 6 -c 1 -o gpurun_out/prof_fibbatch_steady python tools/run_config.py fibbatch --reps 2 > gpurun_out/ncu_s3a.log 2>&1; tail -2 gpurun_out/ncu_s3a.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -c 1 -o gpurun_out/prof_ack34 python tools/run_config.py ackermann:3:4 --reps 1 > gpurun_out/ncu_s3b.log 2>&1; tail -2 gpurun_out/ncu_s3b.log
