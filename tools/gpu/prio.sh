mkdir -p gpurun_out
for pr in 4,3,2,1 1,0,2,2 2,0,1,1 0,0,0,0 3,1,2,2 1,1,2,2; do
PLV_TIER_PRIO=$pr timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 > gpurun_out/bp_$pr.json 2>/dev/null
PLV_TIER_PRIO=$pr timeout 300 python bench.py --no-cpu-baseline --no-louvain --steps 10 --mode uncolored > gpurun_out/bpu_$pr.json 2>/dev/null
done
