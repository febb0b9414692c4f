#!/bin/bash
# after the refcount change: tail traces, phase counters of the run-ahead tail, export phases
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/tail_trace.py fibbatch1 fibbatch > gpurun_out/tail_trace.log 2>&1; echo "tail rc=$?"
timeout 300 python tools/run_config.py fibbatch1 --profile --reps 2 > gpurun_out/phases_fibbatch1.log 2>&1; echo "ph rc=$?"
timeout 300 python tools/run_config.py fibbatch --profile --reps 2 > gpurun_out/phases_fibbatch.log 2>&1; echo "ph rc=$?"
timeout 300 python tools/export_phases.py > gpurun_out/export_phases.log 2>&1; echo "exp rc=$?"
timeout 300 python tools/run_config.py ackermann36 --profile --reps 2 > gpurun_out/phases_ackermann36.log 2>&1; echo "ph rc=$?"
