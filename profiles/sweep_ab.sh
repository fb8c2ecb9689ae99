# A/B of k_sweep variants (scratch/libs/*.so via CA_LIBRARY): C5 4096 scenes, ms per sweep launch
for v in intree ${SWEEP_VARIANTS}; do
  if [ $v = intree ]; then L=""; else L=$PWD/scratch/libs/$v.so; fi
  for r in 1 2; do echo -n "$v: "; CA_LIBRARY=$L python profiles/time_sweep.py 4096 10 | tail -1; done
done
