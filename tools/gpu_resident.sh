cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -x -q -m gpu --timeout 240 --timeout_method thread 2>&1 | tail -3
for c in ackermann36 fib18 reverse16k buildsum22 transform22; do for f in "" "--no-resident"; do timeout 300 python tools/run_config.py $c --reps 2 $f 2>&1 | tail -2 | head -1 | cut -c1-220; done; done
for f in "" "--no-resident"; do for c in fibbatch sortbatch; do timeout 300 python tools/sweep_timeline.py $c $f | cut -c1-100; done; done
