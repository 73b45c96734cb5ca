mkdir -p gpurun_out
timeout 600 python tools/run_trace.py c3_grid --repeat 3 > gpurun_out/rt_c3.txt 2>&1
timeout 900 python tools/run_trace.py c4_chung_lu --repeat 1 > gpurun_out/rt_c4.txt 2>&1
