# after the background phase teardown: full GPU tests, run() profiles, bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "rc=$?" >> gpurun_out/smoke2.log
for c in c2_rmat20 c3_grid c4_chung_lu; do
timeout 300 python tools/run_profile.py $c > gpurun_out/rp2_$c.txt 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_full2.json 2> gpurun_out/bench_full2.err
