mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_full_size.py -x -q --durations=5 > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log
