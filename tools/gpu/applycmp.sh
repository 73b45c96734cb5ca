mkdir -p gpurun_out
for cfg in "8 1024" "4 1024" "16 1024" "8 512" "8 2048"; do
  set -- $cfg
  sed -i "s/^constexpr int64_t APPLY_THREAD_MAX = [0-9]*;/constexpr int64_t APPLY_THREAD_MAX = $1;/" paper_1410_1237_b200/csrc/apply.cu
  sed -i "s/^constexpr int64_t APPLY_HUGE = [0-9]*;/constexpr int64_t APPLY_HUGE = $2;/" paper_1410_1237_b200/csrc/apply.cu
  python -m paper_1410_1237_b200.build > /dev/null 2>&1
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/ap_$1_$2_u_$r.json 2>/dev/null
  done
  timeout 300 python tools/capped_timeline.py c3_grid --phase 4 --iters 5 > gpurun_out/ap_$1_$2_c3.txt 2>&1
done
