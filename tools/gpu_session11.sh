timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_s11.json 2> gpurun_out/bench_s11.err; tail -2 gpurun_out/bench_s11.err; cat gpurun_out/bench_s11.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_s11.json 2>&1; cat gpurun_out/bench_ref_s11.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s11.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > /dev/null 2>&1; grep -c step_loop gpurun_out/launches_s11.csv
nproc; lscpu | grep "Model name"
