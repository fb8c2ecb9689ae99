# A/B of library variants (scratch/libs/*.so via CA_LIBRARY) on the C5 prox_eps=1e-2 sweep
for v in intree ${PROX_VARIANTS}; do
  if [ $v = intree ]; then L=""; else L=$PWD/scratch/libs/$v.so; fi
  CA_LIBRARY=$L python bench.py --prox-eps 1e-2 --no-cpu --no-e2e --steps 3 --warmup 3 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['sweep'])"
done
