# quick check: GPU parity tests + colored/uncolored bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 200 python tools/timeline.py --dump gpurun_out/tl_c.tsv > gpurun_out/tl_c.txt 2>&1
timeout 200 python tools/ktrace.py > gpurun_out/ktrace.txt 2>&1
