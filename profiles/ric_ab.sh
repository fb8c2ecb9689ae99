# A/B of k_riccati_scan variants (scratch/libs/*.so via CA_LIBRARY) on C2 / C4:
# per-iteration solve time, ncu kernel duration, phase cycles (instrumented builds)
mkdir -p gpurun_out/r02
for v in intree ${RIC_VARIANTS:-r_ge}; do
  if [ $v = intree ]; then L=""; else L=$PWD/scratch/libs/$v.so; fi
  echo "== $v"
  for c in 2 4; do CA_LIBRARY=$L python profiles/time_solve.py $c 5; done
  CA_LIBRARY=$L ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/prof_cfg.py 4 10 > gpurun_out/r02/ncu_ric_$v.csv 2>/dev/null
  python profiles/ncu_sum.py gpurun_out/r02/ncu_ric_$v.csv | grep -o "'void k_riccati[^)]*)"
done
for v in ${RIC_PROF:-r_prof r_profge}; do echo "== $v"; CA_LIBRARY=$PWD/scratch/libs/$v.so python profiles/prof_cfg.py 4 2 | grep -E "cycles" | tail -2; done
timeout 900 python -m pytest tests/test_gpu_riccati.py tests/test_gpu_parity.py tests/test_gpu_closed_loop.py tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider -k "riccati or t1_primal or t2_full or closed or box or solve_parity" 2>&1 | tail -3
