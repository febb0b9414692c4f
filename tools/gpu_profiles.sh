#!/bin/bash
# round profiles: bench line, launch list of the bench command, ncu --set full of the top kernels
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-gate > /dev/null 2>&1; echo "launches rc=$?"
for c in fibbatch sortbatch buildsum22; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_loop -s 1 -c 1 \
      -o gpurun_out/ncu_$c python tools/profile_target.py $c > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:export_store -c 1 \
    -o gpurun_out/ncu_export python tools/e2e_parts.py > gpurun_out/ncu_export.log 2>&1; echo "ncu export rc=$?"
