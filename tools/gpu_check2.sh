cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multirank.py tests/test_gpu_dropin.py -q --timeout 300 > gpurun_out/pytest_part.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_part.log
tail -3 gpurun_out/pytest_part.log
bash tools/sanitize.sh
