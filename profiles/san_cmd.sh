set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python profiles/sanitize.py c2 > gpurun_out/san/plain_c2.log 2>&1; echo "plain c2 rc=$?"
python profiles/sanitize.py c5 32 > gpurun_out/san/plain_c5.log 2>&1; echo "plain c5 rc=$?"
python profiles/time_sweep.py 4096 10 > gpurun_out/san/time_sweep_base.log 2>&1; echo "time rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 500 compute-sanitizer --tool $tool --print-limit 40 python profiles/sanitize.py c2 > gpurun_out/san/${tool}_c2.log 2>&1; echo "$tool c2 rc=$?"
  timeout 700 compute-sanitizer --tool $tool --print-limit 40 python profiles/sanitize.py c5 32 > gpurun_out/san/${tool}_c5.log 2>&1; echo "$tool c5 rc=$?"
done
tail -n 3 gpurun_out/san/*.log
