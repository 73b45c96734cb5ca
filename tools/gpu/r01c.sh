# Round-1 final evidence: tests, smoke, bench (both arms), uncoloured line,
# other configs, torchrun + partitioned plumbing, launch list, per-iteration
# DRAM summaries, timelines, run() profiles, full captures of two kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
for c in c1_sbm c3_grid c4_chung_lu; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-louvain --partitioned > gpurun_out/torchrun_part.json 2> gpurun_out/torchrun_part.err; echo "rc=$?" >> gpurun_out/torchrun_part.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-louvain \
  > gpurun_out/ncu_launch.log 2>&1
for m in colored uncolored; do
timeout 600 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iter_$m.csv python tools/profile_iter.py --mode $m > gpurun_out/pi_$m.log 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterw_$m.csv python tools/profile_iter.py --mode $m > gpurun_out/piw_$m.log 2>&1
done
timeout 900 ncu --profile-from-start off -k regex:k_decide_t2 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/t2_full python tools/profile_iter.py --mode uncolored \
  > gpurun_out/t2_full.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_hub_pass -s 100 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/hubpass_full python tools/profile_iter.py --mode colored \
  > gpurun_out/hubpass_full.log 2>&1
timeout 600 python tools/timeline.py --dump gpurun_out/tl_c.tsv > gpurun_out/tl_c.txt 2>&1
timeout 600 python tools/timeline.py --mode uncolored --dump gpurun_out/tl_u.tsv > gpurun_out/tl_u.txt 2>&1
for c in c2_rmat20 c3_grid c4_chung_lu; do
timeout 300 python tools/run_profile.py $c > gpurun_out/rp_$c.txt 2>&1
done
timeout 300 python tools/capped_timeline.py c3_grid --phase 4 > gpurun_out/ct_c3p4.txt 2>&1
timeout 300 python tools/color_timeline.py c4_chung_lu > gpurun_out/colt.txt 2>&1
for c in c4_chung_lu c2_rmat20; do timeout 600 python tools/color_calls.py $c > gpurun_out/colcalls_$c.txt 2>&1; done
timeout 300 python tools/color_timeline_k.py c4_chung_lu 3 > gpurun_out/colt_k3.txt 2>&1
