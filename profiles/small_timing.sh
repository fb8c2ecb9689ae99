# per-iteration latency of the single-scene configs, parallel-in-time primal step vs the serial recursion
for cfg in 1 2 3 4 8 11; do
  python profiles/time_solve.py $cfg 5
  CA_RICCATI_SCAN=0 python profiles/time_solve.py $cfg 5 | sed 's/^/serial: /'
  python profiles/prof_cfg.py $cfg 20 | sed 's/^/scan kernels: /'
  CA_RICCATI_SCAN=0 python profiles/prof_cfg.py $cfg 20 | sed 's/^/serial kernels: /'
done
