# compute-sanitizer memcheck / racecheck / synccheck of the whole pipeline
# (CSR build, VF, colouring, coloured + uncoloured local moving, rebuilds,
# run()) on two small graphs.  Summaries -> gpurun_out/sanitizer_*.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_run.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_$tool.txt
done
