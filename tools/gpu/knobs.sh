mkdir -p gpurun_out
run() {  # name
  python -m paper_1410_1237_b200.build > gpurun_out/kn_$1.build 2>&1 || { echo "build failed $1" > gpurun_out/kn_$1.txt; return; }
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/kn_$1_c2_$r.json 2>/dev/null
  done
  timeout 300 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/kn_$1_c4.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/kn_$1_u.json 2>/dev/null
}
D=paper_1410_1237_b200/csrc/decide.cu
L=paper_1410_1237_b200/csrc/localmove.cuh
run base
sed -i 's/^constexpr int T2_WIDE_MAX = 148;/constexpr int T2_WIDE_MAX = 64;/' $D; run wide64
sed -i 's/^constexpr int T2_WIDE_MAX = 64;/constexpr int T2_WIDE_MAX = 400;/' $D; run wide400
sed -i 's/^constexpr int T2_WIDE_MAX = 400;/constexpr int T2_WIDE_MAX = 148;/' $D
sed -i 's/^constexpr int HSB = 512; /constexpr int HSB = 256; /' $D; run hsb256
sed -i 's/^constexpr int HSB = 256; /constexpr int HSB = 512; /' $D
sed -i 's/^constexpr int T1_WARPS = 8;/constexpr int T1_WARPS = 4;/' $L; run t1w4
