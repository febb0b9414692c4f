cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python tools/race_hunt.py 300 '{"disable_warp_mode": 1}' fib12 fib10 ackermann23 > gpurun_out/race1.log 2>&1
python tools/race_hunt.py 300 '{}' fib12 mergesort50_s42 > gpurun_out/race2.log 2>&1
python tools/race_hunt.py 300 '{"disable_warp_mode": 1, "no_runahead": 1}' fib12 > gpurun_out/race3.log 2>&1
python tools/race_hunt.py 300 '{"disable_warp_mode": 1, "no_resident": 1}' fib12 > gpurun_out/race4.log 2>&1
