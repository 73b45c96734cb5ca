# Round-2 evidence pass: full GPU suite, reference suite, both bench arms, the
# C4 launch list and per-kernel DRAM traffic (warm caches), timelines, a full
# ncu capture of the top C4 kernel.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for m in colored uncolored; do
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterw_c4_$m.csv python tools/profile_iter.py --config c4_chung_lu --mode $m > gpurun_out/piw_c4_$m.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-louvain \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_decide_t0 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_t0_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_t0_full.log 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
timeout 600 python tools/timeline.py --config c2_rmat20 > gpurun_out/tl_c2c.txt 2>&1
timeout 600 python tools/timeline.py --config c2_rmat20 --mode uncolored > gpurun_out/tl_c2u.txt 2>&1
for c in c2_rmat20 c3_grid c4_chung_lu; do timeout 300 python tools/run_profile.py $c > gpurun_out/rp_$c.txt 2>&1; done
