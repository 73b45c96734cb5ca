mkdir -p gpurun_out
timeout 300 python tools/run_profile.py c2_rmat20 > gpurun_out/rp_c2.txt 2>&1
timeout 300 python tools/run_profile.py c2_rmat20 --bench-like > gpurun_out/rp_c2b.txt 2>&1
timeout 300 python tools/run_profile.py c3_grid > gpurun_out/rp_c3.txt 2>&1
