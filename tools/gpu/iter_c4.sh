mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --csv \
  --log-file gpurun_out/iter_c4u.csv python tools/profile_iter.py --config c4_chung_lu --mode uncolored > gpurun_out/pi_c4u.log 2>&1
