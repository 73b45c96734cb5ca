mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.used,memory.total --format=csv > gpurun_out/mem.txt
timeout 900 python bench.py --scale 24 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s24.json 2> gpurun_out/bench_s24.err
echo "rc=$?" >> gpurun_out/bench_s24.err
timeout 1200 python bench.py --scale 26 --steps 3 --warmup 3 --no-cpu-baseline --no-louvain > gpurun_out/bench_s26.json 2> gpurun_out/bench_s26.err
echo "rc=$?" >> gpurun_out/bench_s26.err
