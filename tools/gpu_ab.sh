#!/bin/bash
# knob A/B on one B200: KNOBS (json list of env dicts) over the configs given
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
out=gpurun_out/${AB_OUT:-ab}.log
timeout ${AB_TIMEOUT:-1500} python tools/knob_ab.py "$@" > $out 2>&1; echo "ab rc=$?" >> $out
tail -40 $out
