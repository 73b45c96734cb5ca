mkdir -p gpurun_out
F=paper_1410_1237_b200/csrc/color.cu
cp $F /tmp/color_base.cu
for C in 2048 1024; do
  sed -i "s/^constexpr int64_t CHUGE = [0-9]*;/constexpr int64_t CHUGE = $C;/" $F
  python -m paper_1410_1237_b200.build > gpurun_out/ch_$C.build 2>&1
  timeout 600 python -m pytest tests -m gpu -x -q -k "color or colour or full_size" > gpurun_out/ch_${C}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ch_${C}_tests.log
  for c in c4_chung_lu c2_rmat20 c3_grid; do timeout 600 python tools/color_calls.py $c > gpurun_out/ch_${C}_$c.txt 2>&1; done
done
cp /tmp/color_base.cu $F
python -m paper_1410_1237_b200.build > /dev/null 2>&1
