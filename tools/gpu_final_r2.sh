#!/bin/bash
# round-2 closing measurements: bench line, reference arm, launch list, ncu --set full of the step loop per config,
# then compute-sanitizer over the changed publication protocol
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/*
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-gate > /dev/null 2>&1; echo "launches rc=$?"
for c in fibbatch fibbatch1 fib18 transform22 buildsum22 sortbatch; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:step_loop -c 4 \
      -o /tmp/ncu/ncu_$c python tools/profile_target.py $c > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
cp profiles/traffic.json gpurun_out/traffic_before.json
python tools/ncu_summary.py /tmp/ncu r2 gpurun_out > gpurun_out/ncu_summary.log 2>&1; echo "summary rc=$?"
SAN_TIMEOUT=600 bash tools/sanitize.sh
