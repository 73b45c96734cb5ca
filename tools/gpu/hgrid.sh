mkdir -p gpurun_out
F=paper_1410_1237_b200/csrc/color.cu
cp $F /tmp/color_base.cu
for G in 8 3 16; do
  sed -i "s/^constexpr unsigned HUGE_GRID_MAX = 148 \* [0-9]*;/constexpr unsigned HUGE_GRID_MAX = 148 * $G;/" $F
  python -m paper_1410_1237_b200.build > /dev/null 2>&1
  for c in c4_chung_lu c2_rmat20; do timeout 600 python tools/color_calls.py $c > gpurun_out/hg_${G}_$c.txt 2>&1; done
done
cp /tmp/color_base.cu $F
python -m paper_1410_1237_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "color or colour or full_size or parity" > gpurun_out/colq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/colq_tests.log
