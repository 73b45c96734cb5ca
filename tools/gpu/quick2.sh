mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
for c in c4_chung_lu c3_grid; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-louvain > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_${c}_u.json 2> gpurun_out/bench_${c}_u.err
done
