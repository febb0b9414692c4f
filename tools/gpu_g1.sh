cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu --timeout 300 > gpurun_out/fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize.log
tail -5 gpurun_out/fullsize.log
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 240 --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
