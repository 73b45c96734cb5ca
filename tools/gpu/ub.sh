mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-louvain --mode uncolored --steps 5 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
timeout 200 python tools/timeline.py --mode uncolored --dump gpurun_out/tl_u.tsv > gpurun_out/tl_u.txt 2>&1
timeout 300 python tools/capped_timeline.py c4_chung_lu --phase 5 > gpurun_out/ct_c4p5.txt 2>&1
