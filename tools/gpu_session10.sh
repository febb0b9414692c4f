timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_s10.json 2> gpurun_out/bench_s10.err; tail -2 gpurun_out/bench_s10.err; cat gpurun_out/bench_s10.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s10.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > /dev/null 2>&1; grep -c step_loop gpurun_out/launches_s10.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 1 -c 1 -o gpurun_out/prof_fibbatch_s10 python tools/profile_target.py fibbatch > gpurun_out/ncu_s10a.log 2>&1; tail -3 gpurun_out/ncu_s10a.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 1 -c 1 -o gpurun_out/prof_sortbatch_s10 python tools/profile_target.py sortbatch > gpurun_out/ncu_s10b.log 2>&1; tail -3 gpurun_out/ncu_s10b.log
