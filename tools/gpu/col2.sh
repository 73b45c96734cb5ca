mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "color or golden or run" > gpurun_out/col_tests.log 2>&1; echo "rc=$?" >> gpurun_out/col_tests.log
timeout 300 python tools/color_timeline.py c4_chung_lu > gpurun_out/colt_c4.txt 2>&1
timeout 300 python tools/color_timeline.py c2_rmat20 > gpurun_out/colt_c2.txt 2>&1
timeout 300 python tools/run_profile.py c2_rmat20 > gpurun_out/rp_c2.txt 2>&1
