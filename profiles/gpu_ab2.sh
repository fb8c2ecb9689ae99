# A/B sweep timings (two alternations to see box noise) then the parity tiers
mkdir -p gpurun_out/r02
for r in 1 2; do python profiles/tune.py time 4096 10; done > gpurun_out/r02/ab.log 2>&1; cat gpurun_out/r02/ab.log | cut -c1-160
timeout 1800 python -m pytest ${PYTEST_ARGS:-tests -m gpu} -x -q -p no:cacheprovider > gpurun_out/r02/gpu_tests.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^E |^FAILED" gpurun_out/r02/gpu_tests.log | cut -c1-300 | tail -12
