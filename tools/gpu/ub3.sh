mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored --steps 5 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 200 python tools/timeline.py --mode uncolored --dump gpurun_out/tl_u.tsv > gpurun_out/tl_u.txt 2>&1
