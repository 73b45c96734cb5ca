mkdir -p gpurun_out
run() {
  python -m paper_1410_1237_b200.build > gpurun_out/ck_$1.build 2>&1 || { echo "build failed" > gpurun_out/ck_$1.txt; return; }
  timeout 300 python tools/color_timeline.py c4_chung_lu > gpurun_out/ck_$1_c4.txt 2>&1
  timeout 300 python tools/color_timeline.py c2_rmat20 > gpurun_out/ck_$1_c2.txt 2>&1
}
C=paper_1410_1237_b200/csrc/color.cu
run base
sed -i 's/^constexpr int64_t CMID_MAXD = 512;/constexpr int64_t CMID_MAXD = 256;/' $C; run mid256
sed -i 's/^constexpr int64_t CMID_MAXD = 256;/constexpr int64_t CMID_MAXD = 1024;/' $C; run mid1024
sed -i 's/^constexpr int64_t CMID_MAXD = 1024;/constexpr int64_t CMID_MAXD = 512;/' $C
sed -i 's/^constexpr int COLOR_THREAD_MAXD = 32;/constexpr int COLOR_THREAD_MAXD = 16;/' $C; run thr16
sed -i 's/^constexpr int COLOR_THREAD_MAXD = 16;/constexpr int COLOR_THREAD_MAXD = 64;/' $C; run thr64
