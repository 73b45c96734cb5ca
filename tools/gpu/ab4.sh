mkdir -p gpurun_out
rm -f gpurun_out/ab_summary.txt
for v in ${VARS:-_ trig u4 u4trig u4b3}; do
  [ "$v" = "_" ] && vv="" || vv=$v
  tag=${v}
  PLV_VARIANT=$vv timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-louvain \
      > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$tag.json')); print('$v', round(d['ms_per_step'],3),'ms', 'decide', round(d['roofline']['ms_per_iter'],3), 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/ab_summary.txt 2>&1
done
