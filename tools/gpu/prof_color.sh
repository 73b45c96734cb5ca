# ncu --set full of the huge-row colouring kernels on C4's first colouring
mkdir -p gpurun_out
for K in k_color_assign_huge k_color_conflicts_huge; do
timeout 900 ncu -k "regex:$K" -s 40 -c 2 --set full --import-source on \
  --clock-control none -f -o gpurun_out/col_$K python tools/color_timeline.py c4_chung_lu \
  > gpurun_out/col_$K.log 2>&1
echo "rc=$?" >> gpurun_out/col_$K.log
done
