#!/bin/bash
# round-2 profiles: bench line, reference arm, launch list, ncu --set full of the step loop per config and of
# the export, canonical relabelling and gather probe kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/*
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-gate > /dev/null 2>&1; echo "launches rc=$?"
for c in fibbatch transform22 fib18 sortbatch buildsum22 fibbatch1; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:step_loop -c 4 \
      -o /tmp/ncu/ncu_$c python tools/profile_target.py $c > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:export_store -c 1 \
    -o /tmp/ncu/ncu_export python tools/e2e_parts.py > gpurun_out/ncu_export.log 2>&1; echo "ncu export rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:canon_down -c 1 \
    -o /tmp/ncu/ncu_canon python tools/canon_target.py > gpurun_out/ncu_canon.log 2>&1; echo "ncu canon rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:gather_probe -s 1 -c 1 \
    -o /tmp/ncu/ncu_probe python tools/probe_target.py > gpurun_out/ncu_probe.log 2>&1; echo "ncu probe rc=$?"
timeout 600 python tools/layout_ab.py > gpurun_out/layout_ab.log 2>&1; timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:probe_ --csv --log-file gpurun_out/ncu_layout.csv python tools/layout_ab.py > gpurun_out/ncu_layout.log 2>&1; echo "layout rc=$?"

# summaries only (the .ncu-rep files stay on the box: gpurun_out is capped at 64 MiB)
python tools/ncu_summary.py /tmp/ncu r2 gpurun_out > gpurun_out/ncu_summary.log 2>&1; echo "summary rc=$?"
for f in /tmp/ncu/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > gpurun_out/${b}_details.csv 2>/dev/null
done
ls -la gpurun_out | tail -40
# run-ahead on/off per config, and the phase cycle accounting of the latency-bound chains
timeout 900 python tools/ra_compare.py > gpurun_out/ra_compare.log 2>&1; echo "ra_compare rc=$?"
for c in ackermann36 fib18 reverse16k; do
  timeout 300 python tools/run_config.py $c --profile --reps 2 > gpurun_out/phases_$c.log 2>&1; echo "phases $c rc=$?"
done
