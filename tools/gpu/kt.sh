mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ahead.py -x -q > gpurun_out/ahead_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ahead_tests.log
for c in 10 12 16 20 24; do
PLV_AHEAD_CAP8=$c timeout 900 python bench.py --no-cpu-baseline --no-louvain > gpurun_out/bench_cap$c.json 2> gpurun_out/bench_cap$c.err
done
