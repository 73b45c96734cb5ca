# quick A/B on the coloured C2 / C4 iteration only: tools/gpu/ab2.sh "v1 v2 ..."
mkdir -p gpurun_out
for v in $1; do
  [ "$v" = "_" ] && vv="" || vv=$v
  for cfg in c4_chung_lu c2_rmat20; do
    PLV_VARIANT=$vv timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-louvain \
      > gpurun_out/ab2_${v}_$cfg.json 2> gpurun_out/ab2_${v}_$cfg.err
    python -c "import json; d=json.load(open('gpurun_out/ab2_${v}_$cfg.json')); print('$v','$cfg', round(d['ms_per_step'],3),'ms')" >> gpurun_out/ab_summary.txt 2>&1
  done
done
