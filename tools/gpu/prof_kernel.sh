# usage: bash tools/gpu/prof_kernel.sh <kernel-regex> <out-name> [mode] [count]
K=$1; OUT=$2; MODE=${3:-colored}; C=${4:-3}
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off -k "regex:$K" -c $C --set full --import-source on \
  --clock-control none --warp-sampling-interval 0 -f -o gpurun_out/$OUT python tools/profile_iter.py --mode $MODE \
  > gpurun_out/$OUT.log 2>&1
echo "rc=$?" >> gpurun_out/$OUT.log
