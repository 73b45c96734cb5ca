mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_golden.py tests/test_full_size.py -x -q > gpurun_out/t0_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t0_tests.log
for v in _ nofilt; do
[ "$v" = "_" ] && vv="" || vv=$v
PLV_VARIANT=$vv timeout 900 python bench.py --no-cpu-baseline --no-louvain > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
PLV_VARIANT=$vv timeout 900 python bench.py --config c2_rmat20 --no-cpu-baseline --no-louvain > gpurun_out/bench_c2_$v.json 2> gpurun_out/bench_c2_$v.err
PLV_VARIANT=$vv timeout 900 python bench.py --config c4_chung_lu --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_c4u_$v.json 2> gpurun_out/bench_c4u_$v.err
done
timeout 600 python tools/timeline.py --config c4_chung_lu > gpurun_out/tl_c4c.txt 2>&1
