mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored --steps 10 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 600 python tools/run_trace.py c3_grid --repeat 1 > gpurun_out/rt_c3.txt 2>&1
