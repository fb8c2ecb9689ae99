# kernel durations of the single-scene configs (ncu launch list), scan vs serial primal step
mkdir -p gpurun_out/r02
for cfg in 2 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/prof_cfg.py $cfg 10 > gpurun_out/r02/ncu_small_c${cfg}_scan.csv 2>/dev/null
  CA_RICCATI_SCAN=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/prof_cfg.py $cfg 10 > gpurun_out/r02/ncu_small_c${cfg}_serial.csv 2>/dev/null
done
