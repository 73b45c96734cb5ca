mkdir -p gpurun_out
for c in c4_chung_lu c3_grid c1_sbm; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_${c}_u.json 2> gpurun_out/bench_${c}_u.err
done
