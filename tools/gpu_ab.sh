# same-box A/B of the working build against tools/variants/prev.so (+ GPU tests of the working build)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for v in tools/variants/prev.so "" tools/variants/prev.so ""; do
  SD_LIB_OVERRIDE=$v timeout 300 python bench.py --no-cpu-baseline --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/ab.json
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('${v:-new}', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done
