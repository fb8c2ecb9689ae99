# one GPU call: build check, the GPU test tiers, a quick sweep timing
set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/r02/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02/gpu_tests.log
python profiles/time_sweep.py 4096 10 > gpurun_out/r02/time_sweep.log 2>&1; cat gpurun_out/r02/time_sweep.log
