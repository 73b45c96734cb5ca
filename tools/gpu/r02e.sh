# Re-entry validation: GPU suite, smoke, default bench, C4 timeline dump, stage stats.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c.tsv > gpurun_out/tl_c4c.txt 2>&1
timeout 600 python tools/stage_stats.py c4_chung_lu > gpurun_out/stage_stats_c4.txt 2>&1
