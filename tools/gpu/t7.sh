mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 600 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c3_grid --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
