# Round-2 evidence for the final code (ahead tables): GPU suite (default, and
# with low-degree stages forced through the ahead path), smoke, both bench arms
# (C4 headline), context lines, warm-cache DRAM traffic of the C4 iterations,
# launch list, timelines, per-block trace of the ahead pass, run() profiles,
# full captures of the ahead pass / accumulation and the tier-0 decide.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
PLV_AHEAD_LOWDEG=1 timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_lowdeg.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_lowdeg.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
PLV_AHEAD=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_noahead.json 2> gpurun_out/bench_noahead.err
timeout 600 python bench.py --mode uncolored --no-cpu-baseline > gpurun_out/bench_c4u.json 2> gpurun_out/bench_c4u.err
for c in c2_rmat20 c3_grid c1_sbm; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --config c2_rmat20 --mode uncolored --no-cpu-baseline --no-louvain > gpurun_out/bench_c2u.json 2> gpurun_out/bench_c2u.err
for m in colored uncolored; do
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterw_c4_$m.csv python tools/profile_iter.py --config c4_chung_lu --mode $m > gpurun_out/piw_c4_$m.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-louvain \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_ah_pass -s 250 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_ah_pass_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_ah_pass_full.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_ah_accum -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_ah_accum_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_ah_accum_full.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_decide_t0 -s 1 -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4_t0_stage1_full python tools/profile_iter.py --config c4_chung_lu \
  > gpurun_out/c4_t0_stage1_full.log 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --mode uncolored > gpurun_out/tl_c4u.txt 2>&1
timeout 600 python tools/timeline.py --config c2_rmat20 > gpurun_out/tl_c2c.txt 2>&1
KTRACE_ON=2 timeout 600 python tools/ktrace.py colored c4_chung_lu > gpurun_out/ktrace_c4_ah.txt 2>&1
for c in c2_rmat20 c3_grid c4_chung_lu; do timeout 300 python tools/run_profile.py $c > gpurun_out/rp_$c.txt 2>&1; done
timeout 300 python tools/run_kernels.py c4_chung_lu 30 > gpurun_out/rk_c4.txt 2>&1
timeout 300 python tools/ahead_stats.py c4_chung_lu > gpurun_out/ahead_stats_c4.txt 2>&1
[ -x tools/l2_gather ] && tools/l2_gather > gpurun_out/l2_gather.txt 2>&1
timeout 300 python tools/capped_timeline.py c3_grid --phase 4 > gpurun_out/capped_c3_p4.txt 2>&1
