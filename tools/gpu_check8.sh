#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dropin.py -x -q -m gpu -k "export or fetch or canonical or dropin or store or refcount" > gpurun_out/t_export.log 2>&1; echo "t rc=$?"
timeout 300 python tools/export_phases.py > gpurun_out/export_phases.log 2>&1; echo "exp rc=$?"
KNOBS='[{}, {"TRS_B200_JIT_DEFINES": "-DTRS_B200_RA_PREFETCH=0"}]' timeout 900 python tools/knob_ab.py fibbatch fib18 reverse16k ackermann36 > gpurun_out/knob_prefetch2.log 2>&1; echo "knob rc=$?"
