mkdir -p gpurun_out
tools/l2_gather > gpurun_out/l2_gather.txt 2>&1
timeout 900 python -m pytest tests/test_ahead.py -x -q > gpurun_out/ahead_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ahead_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
