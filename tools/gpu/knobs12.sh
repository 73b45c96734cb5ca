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
L=paper_1410_1237_b200/csrc/localmove.cuh
run blk512b
sed -i 's/^constexpr int BLK = 512; /constexpr int BLK = 1024; /' $L; run blk1024
