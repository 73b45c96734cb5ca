# end-of-session check: full GPU tests, smoke, default bench line, colouring and run() evidence
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench_full.json 2> gpurun_out/f_bench_full.err
timeout 600 python bench.py --config c4_chung_lu --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
for c in c4_chung_lu c2_rmat20; do timeout 600 python tools/color_calls.py $c > gpurun_out/f_colcalls_$c.txt 2>&1; done
timeout 300 python tools/color_timeline.py c4_chung_lu > gpurun_out/f_colt.txt 2>&1
timeout 300 python tools/color_timeline_k.py c4_chung_lu 3 > gpurun_out/f_colt_k3.txt 2>&1
for c in c2_rmat20 c4_chung_lu; do timeout 300 python tools/run_profile.py $c > gpurun_out/f_rp_$c.txt 2>&1; done
