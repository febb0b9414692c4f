timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -m gpu 2>&1 | tail -2
TRS_B200_RICH_ENTRIES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for v in 1 2; do for c in fibbatch sortbatch transform22 buildsum22; do timeout 120 python tools/run_config.py $c --reps 2 --variant $v 2>&1 | tail -2 | head -1; done; done
for c in fibbatch sortbatch; do TRS_B200_RICH_ENTRIES=1 timeout 120 python tools/run_config.py $c --reps 2 --variant 2 2>&1 | tail -2 | head -1; done
