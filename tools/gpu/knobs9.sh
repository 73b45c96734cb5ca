mkdir -p gpurun_out
run() {  # name
  python -m paper_1410_1237_b200.build > gpurun_out/kn_$1.build 2>&1 || { echo "build failed $1" > gpurun_out/kn_$1.txt; return; }
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/kn_$1_c2_$r.json 2>/dev/null
  done
  timeout 300 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/kn_$1_c4.json 2>/dev/null
  for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/kn_$1_u_$r.json 2>/dev/null
  done
}
A=paper_1410_1237_b200/csrc/apply.cu
run base9
sed -i 's/^constexpr int APPLY_BB = 148 \* 8;/constexpr int APPLY_BB = 148 * 16;/' $A; run bb16
sed -i 's/^constexpr int APPLY_BB = 148 \* 16;/constexpr int APPLY_BB = 148 * 4;/' $A; run bb4
sed -i 's/^constexpr int APPLY_BB = 148 \* 4;/constexpr int APPLY_BB = 148 * 8;/' $A
sed -i 's/^constexpr int APPLY_HB = 148 \* 4;/constexpr int APPLY_HB = 148 * 2;/' $A; run hb2
