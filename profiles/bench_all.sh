# the bench lines of this round (one B200): default C5, C1-C4, the reference arm
mkdir -p gpurun_out/r02
python bench.py > gpurun_out/r02/bench_c5.json 2> gpurun_out/r02/bench_c5.err; echo "c5 rc=$?"
for c in 1 2 3 4; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r02/bench_c$c.json 2> gpurun_out/r02/bench_c$c.err; echo "c$c rc=$?"; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02/bench_ref.json 2> gpurun_out/r02/bench_ref.err; echo "ref rc=$?"
python bench.py --prox-eps 1e-2 --no-cpu > gpurun_out/r02/bench_c5_prox.json 2> gpurun_out/r02/bench_c5_prox.err; echo "prox rc=$?"
