mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "color or colour or full_size or parity" > gpurun_out/colq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/colq_tests.log
for c in c4_chung_lu c2_rmat20 c3_grid; do timeout 600 python tools/color_calls.py $c > gpurun_out/cc2_$c.txt 2>&1; done
