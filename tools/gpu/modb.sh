mkdir -p gpurun_out
python tools/mod_bench.py > gpurun_out/modb.txt 2>&1
timeout 300 ncu -k regex:k_mod_fused -c 2 --set full --import-source on -f -o gpurun_out/modf python tools/mod_bench.py 1573370 > gpurun_out/modf.log 2>&1
