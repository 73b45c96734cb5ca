# tier-boundary sweep: T1_MAXD, T2A_MAXD (+T2A_TS), T2_MAXD (+T2_TS)
mkdir -p gpurun_out
L=paper_1410_1237_b200/csrc/localmove.cuh
cp $L /tmp/lm_base.cuh
run() {  # name
  python -m paper_1410_1237_b200.build > gpurun_out/kn_$1.build 2>&1 || { echo "build failed $1" > gpurun_out/kn_$1.txt; return; }
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/kn_$1_c2_$r.json 2>/dev/null
  done
  timeout 300 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/kn_$1_c4.json 2>/dev/null
  for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/kn_$1_u_$r.json 2>/dev/null
  done
  cp /tmp/lm_base.cuh $L
}
run base13
sed -i 's/^constexpr int T1_MAXD = 128;/constexpr int T1_MAXD = 64;/' $L; run t1_64
sed -i 's/^constexpr int T1_MAXD = 128;/constexpr int T1_MAXD = 96;/' $L; run t1_96
sed -i 's/^constexpr int T2A_MAXD = 680;/constexpr int T2A_MAXD = 400;/' $L; run t2a_400
sed -i 's/^constexpr int T2A_MAXD = 680;/constexpr int T2A_MAXD = 1300;/; s/^constexpr int T2A_TS = 1024;/constexpr int T2A_TS = 2048;/' $L; run t2a_1300
sed -i 's/^constexpr int T2_MAXD = 2048;/constexpr int T2_MAXD = 4096;/; s/^constexpr int T2_TS = 4096;/constexpr int T2_TS = 8192;/' $L; run t3_4096
sed -i 's/^constexpr int T2_MAXD = 2048;/constexpr int T2_MAXD = 1024;/' $L; run t3_1024
python -m paper_1410_1237_b200.build > /dev/null 2>&1
