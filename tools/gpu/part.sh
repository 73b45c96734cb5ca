mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partitioned.py tests/test_gpu_parity.py -x -q > gpurun_out/part_tests.log 2>&1; echo "rc=$?" >> gpurun_out/part_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
