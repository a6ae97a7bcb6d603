# compute-sanitizer passes over the product-shape decode (logs -> gpurun_out/)
mkdir -p gpurun_out
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_case.py 6 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
