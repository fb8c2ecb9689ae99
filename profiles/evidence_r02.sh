# Round-2 evidence on one B200: GPU tests, smoke, bench lines, ncu launch list of the bench
# command, one ncu --set full of the full-size C5 sweep (traffic)
set -x
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02/gpu_tests_final.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02/gpu_tests_final.log
python __graft_entry__.py smoke > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc=$?"
bash profiles/bench_all.sh
python profiles/pivot_hist.py --gpu > gpurun_out/r02/pivot_hist.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02/launches_bench_c5.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02/ncu_launches.log 2>&1; echo "ncu list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_sweep --launch-skip 2 --launch-count 1 -o gpurun_out/r02/sweep_full_c5_r02 python profiles/prof_full.py > gpurun_out/r02/ncu_full.log 2>&1; echo "ncu full rc=$?"
