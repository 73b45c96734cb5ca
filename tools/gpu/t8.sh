mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for r in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/bench_c_$r.json 2>/dev/null; done
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored --steps 10 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 600 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c3_grid --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python tools/run_trace.py c3_grid --repeat 1 > gpurun_out/rt_c3.txt 2>&1
