set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
