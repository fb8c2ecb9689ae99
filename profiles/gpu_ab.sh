# A/B timing of tuning variants (scratch/libs) and the in-tree library, then GPU tests
set -x
mkdir -p gpurun_out/r02
python profiles/tune.py time 4096 10 > gpurun_out/r02/ab.log 2>&1; cat gpurun_out/r02/ab.log
python profiles/time_sweep.py 4096 10 >> gpurun_out/r02/ab.log 2>&1; tail -1 gpurun_out/r02/ab.log
timeout 1800 python -m pytest ${PYTEST_ARGS:-tests -m gpu} -x -q -s -p no:cacheprovider > gpurun_out/r02/gpu_tests.log 2>&1; echo "pytest rc=$?"
grep -E "C5|iterations|passed|failed|Error|error" gpurun_out/r02/gpu_tests.log | tail -30
