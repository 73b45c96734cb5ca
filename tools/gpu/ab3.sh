# A/B of ahead variants on the C4 coloured iteration: build variants x window slots.
mkdir -p gpurun_out
rm -f gpurun_out/ab_summary.txt
for v in _ trig minb4 trigminb; do
  [ "$v" = "_" ] && vv="" || vv=$v
  for sl in 0 4194304 16777216; do
    tag=${v}_$sl
    PLV_AHEAD_SLOTS=$sl PLV_VARIANT=$vv timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-louvain \
      > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_$tag.json')); print('$v','$sl', round(d['ms_per_step'],3),'ms', 'decide', round(d['roofline']['ms_per_iter'],3), 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/ab_summary.txt 2>&1
  done
done
PLV_AHEAD_SLOTS=4194304 timeout 600 python tools/timeline.py --config c4_chung_lu --dump gpurun_out/tl_c4c_4m.tsv > gpurun_out/tl_c4c_4m.txt 2>&1
