mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ahead.py -x -q > gpurun_out/ahead_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ahead_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
PLV_AHEAD_LOWDEG=1 PLV_AHEAD_WIN0=20000 PLV_AHEAD_WIN=50000 timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_lowdeg.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_lowdeg.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
