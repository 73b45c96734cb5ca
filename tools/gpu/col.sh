mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "color or vf or run or golden" > gpurun_out/col_tests.log 2>&1; echo "rc=$?" >> gpurun_out/col_tests.log
for t in 0 256 1024 8192; do
PLV_COLOR_TAIL=$t timeout 300 python tools/run_profile.py c2_rmat20 > gpurun_out/rp_c2_$t.txt 2>&1
PLV_COLOR_TAIL=$t timeout 300 python tools/run_profile.py c4_chung_lu > gpurun_out/rp_c4_$t.txt 2>&1
done
