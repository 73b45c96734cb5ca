# Round-2 first GPU pass: GPU suite, bench (C4 headline), C4 timelines and
# per-iteration DRAM traffic of the decide kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
timeout 600 python tools/timeline.py --config c4_chung_lu --mode uncolored > gpurun_out/tl_c4u.txt 2>&1
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterw_c4.csv python tools/profile_iter.py --config c4_chung_lu > gpurun_out/piw_c4.log 2>&1
