# primal-step (k_riccati_scan) evidence: phase cycles (instrumented build), per-iteration
# solve times, ncu launch lists scan vs serial, and the parity tests that cover the path
mkdir -p gpurun_out/r02
CA_LIBRARY=$PWD/scratch/libs/r_prof.so python profiles/prof_cfg.py 4 2 | grep -E "cycles" | tail -2
for c in 2 4 8 11; do python profiles/time_solve.py $c 5; done
bash profiles/ncu_small.sh
for c in 2 4; do python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/r02/ncu_small_c${c}_scan.csv")) if len(r)>10]
h=rows[0]; k=h.index("Kernel Name"); v=h.index("Metric Value")
import collections; d=collections.defaultdict(list)
for r in rows[1:]: d[r[k][:40]].append(float(r[v].replace(",","")))
print("C${c}", {n:(round(sum(x)/len(x)/1e3,1),len(x)) for n,x in d.items()})
PY
done
timeout 900 python -m pytest tests/test_gpu_riccati.py tests/test_gpu_parity.py tests/test_gpu_closed_loop.py -m gpu -q -x -p no:cacheprovider -k "riccati or t1_primal or t2_full or closed or box" 2>&1 | tail -3
