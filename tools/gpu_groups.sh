# verify attention: row groups of a chunk adjacent in launch order (share K/V through L2) vs prev build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -k "tcgen05 or verify or production or engine or graph" > gpurun_out/groups_tests.log 2>&1; tail -1 gpurun_out/groups_tests.log
for v in tools/variants/prev.so ""; do echo "== ${v:-new}"; SD_LIB_OVERRIDE=$v timeout 200 python tools/time_tc.py 2>&1 | tail -4; done
for v in tools/variants/prev.so "" tools/variants/prev.so ""; do
  SD_LIB_OVERRIDE=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --ngram-stress --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/g.json
  python -c "import json; d=json.load(open('gpurun_out/g.json')); print('stress ${v:-new}', round(d['ms_per_step'],3), 'ms', round(d['roofline']['avg_launch_us'],1), 'us attn', d['clocks']['sm_mhz'])"
done
SD_LIB_OVERRIDE= timeout 300 python bench.py --no-cpu-baseline --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/g.json
python -c "import json; d=json.load(open('gpurun_out/g.json')); print('T41 new', round(d['ms_per_step'],3), 'ms', round(d['roofline']['avg_launch_us'],1), 'us attn')"
