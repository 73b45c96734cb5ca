mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_phase_loop.py tests/test_partitioned.py tests/test_gpu_parity.py -x -q > gpurun_out/loop_tests.log 2>&1; echo "rc=$?" >> gpurun_out/loop_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored --steps 5 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 600 python tools/run_trace.py c3_grid --repeat 1 > gpurun_out/rt_c3.txt 2>&1
timeout 600 python tools/run_trace.py c4_chung_lu --repeat 2 > gpurun_out/rt_c4.txt 2>&1
