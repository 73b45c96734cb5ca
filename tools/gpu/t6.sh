mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 300 python tools/run_profile.py c2_rmat20 > gpurun_out/rp_c2.txt 2>&1
