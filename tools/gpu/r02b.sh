mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python oracle/ref_suite.py -q > gpurun_out/ref_suite.log 2>&1; echo "rc=$?" >> gpurun_out/ref_suite.log
( time timeout 1200 python bench.py --impl reference ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
( time timeout 900 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/gpu/sanitize.sh
