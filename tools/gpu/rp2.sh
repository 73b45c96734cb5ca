mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_phase_loop.py tests/test_partitioned.py tests/test_gpu_parity.py -x -q > gpurun_out/loop_tests.log 2>&1; echo "rc=$?" >> gpurun_out/loop_tests.log
timeout 300 python tools/run_profile.py c2_rmat20 > gpurun_out/rp_c2.txt 2>&1
timeout 300 python tools/run_profile.py c3_grid > gpurun_out/rp_c3.txt 2>&1
timeout 300 python tools/run_profile.py c4_chung_lu > gpurun_out/rp_c4.txt 2>&1
