# A/B of library variants: tools/gpu/ab.sh "variant1 variant2 ..." ["bench args"]
# ("" = the default libplv.so).  C4 / C2 coloured and C4 uncoloured lines.
mkdir -p gpurun_out
VARS=${1:-"_ nohint"}
for v in $VARS; do
  [ "$v" = "_" ] && vv="" || vv=$v
  for cfg in "--config c4_chung_lu" "--config c4_chung_lu --mode uncolored" "--config c2_rmat20" "--config c2_rmat20 --mode uncolored"; do
    tag=$(echo "$v $cfg" | tr ' -' '__')
    PLV_VARIANT=$vv timeout 600 python bench.py $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-louvain $2 \
      > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_$tag.json')); print('$v','$cfg', round(d['ms_per_step'],3),'ms', 'decide', round(d['roofline']['ms_per_iter'],3), 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/ab_summary.txt 2>&1
  done
done
