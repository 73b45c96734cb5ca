mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --csv \
  --log-file gpurun_out/iterw_c4u.csv python tools/profile_iter.py --config c4_chung_lu --mode uncolored > gpurun_out/piw_c4u.log 2>&1
for k in k_decide_t0 "k_decide_t2" k_hub_accum k_decide_t1; do
timeout 900 ncu --profile-from-start off -k regex:$k -c 1 --set full --import-source on \
  --clock-control none -f -o gpurun_out/c4u_$k python tools/profile_iter.py --config c4_chung_lu --mode uncolored \
  > gpurun_out/c4u_$k.log 2>&1
done
