#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q -m gpu -k "export or fetch or canonical or dropin or store or refcount or e2e" > gpurun_out/t_export.log 2>&1; echo "t rc=$?"
timeout 300 python tools/export_phases.py > gpurun_out/export_phases.log 2>&1; echo "exp rc=$?"
KNOBS='[{}, {"TRS_B200_RUNAHEAD": "1"}, {"TRS_B200_RUNAHEAD": "1", "TRS_B200_RA_MAX": "9472", "TRS_B200_RA_KILL": "18944", "TRS_B200_RA_STEPS": "8"}]' timeout 1200 python tools/knob_ab.py mergesort16k sortbatch_s1 sortbatch > gpurun_out/knob_w16.log 2>&1; echo "knob rc=$?"
