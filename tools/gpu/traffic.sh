mkdir -p gpurun_out
for m in colored uncolored; do
timeout 600 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/iterwarm_$m.csv python tools/profile_iter.py --mode $m > gpurun_out/piw_$m.log 2>&1
done
