# time tools/time_tc.py under each variant library in tools/variants/
mkdir -p gpurun_out
for v in tools/variants/*.so; do echo "== $v"; SD_LIB_OVERRIDE=$v timeout 120 python tools/time_tc.py 2>&1 | tail -4; done > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
