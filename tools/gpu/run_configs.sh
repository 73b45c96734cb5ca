# end-to-end run() per BASELINE config with the per-phase breakdown
mkdir -p gpurun_out
timeout 300 python tools/run_trace.py c1_sbm --cutoff 0 > gpurun_out/rt_c1.txt 2>&1
timeout 300 python tools/run_trace.py c2_rmat20 > gpurun_out/rt_c2.txt 2>&1
timeout 600 python tools/run_trace.py c3_grid > gpurun_out/rt_c3.txt 2>&1
timeout 900 python tools/run_trace.py c4_chung_lu --repeat 1 > gpurun_out/rt_c4.txt 2>&1
