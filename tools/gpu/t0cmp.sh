mkdir -p gpurun_out
for T in 16 8 12; do
  sed -i "s/^constexpr int T0_MAXD = [0-9]*;/constexpr int T0_MAXD = $T;/" paper_1410_1237_b200/csrc/localmove.cuh
  python -m paper_1410_1237_b200.build > /dev/null 2>&1
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/t0_${T}_c2_$r.json 2>/dev/null
    timeout 300 python bench.py --config c4_chung_lu --no-cpu-baseline --no-louvain --steps 5 > gpurun_out/t0_${T}_c4_$r.json 2>/dev/null
  done
  timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/t0_${T}_u.json 2>/dev/null
done
