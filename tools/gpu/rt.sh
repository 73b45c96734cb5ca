mkdir -p gpurun_out
timeout 300 python tools/run_trace.py c2_rmat20 --repeat 3 > gpurun_out/rt_c2.txt 2>&1
timeout 300 python tools/run_trace.py c1_sbm --cutoff 0 --repeat 3 > gpurun_out/rt_c1.txt 2>&1
