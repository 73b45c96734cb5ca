# Round-2 final evidence: GPU suite, smoke, both bench arms (C4 headline),
# context lines (C2, C3, uncoloured), partitioned 1-rank lines, warm-cache
# DRAM traffic of the C4 iterations, launch list, timelines, run() profiles,
# full captures of the top C4 kernels.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --mode uncolored --no-cpu-baseline > gpurun_out/bench_c4u.json 2> gpurun_out/bench_c4u.err
for c in c2_rmat20 c3_grid c1_sbm; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --config c2_rmat20 --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_c2u.json 2> gpurun_out/bench_c2u.err
for sc in 22 25; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --partitioned --scale $sc --steps 5 --warmup 3 --no-cpu-baseline --no-louvain > gpurun_out/bpart_$sc.json 2> gpurun_out/bpart_$sc.err
done
for m in colored uncolored; do
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterw_c4_$m.csv python tools/profile_iter.py --config c4_chung_lu --mode $m > gpurun_out/piw_c4_$m.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-louvain \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_hub_pass -s 200 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_hubpass_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_hubpass_full.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_single_t0 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_single_t0_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_single_t0_full.log 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --mode uncolored > gpurun_out/tl_c4u.txt 2>&1
timeout 600 python tools/timeline.py --config c2_rmat20 > gpurun_out/tl_c2c.txt 2>&1
timeout 600 python tools/timeline.py --config c2_rmat20 --mode uncolored > gpurun_out/tl_c2u.txt 2>&1
for c in c2_rmat20 c3_grid c4_chung_lu; do timeout 300 python tools/run_profile.py $c > gpurun_out/rp_$c.txt 2>&1; done
timeout 300 python tools/run_kernels.py c4_chung_lu 30 > gpurun_out/rk_c4.txt 2>&1
