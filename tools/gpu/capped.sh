mkdir -p gpurun_out
timeout 300 python tools/capped_timeline.py c3_grid --phase 4 > gpurun_out/ct_c3p4.txt 2>&1
timeout 300 python tools/capped_timeline.py c3_grid --phase 6 > gpurun_out/ct_c3p6.txt 2>&1
timeout 600 python tools/capped_timeline.py c4_chung_lu --phase 5 > gpurun_out/ct_c4p5.txt 2>&1
