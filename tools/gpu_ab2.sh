# draft attention one-round merge: kernel tests, draft_bench, same-box step A/B vs tools/variants/prev.so
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -k "draft or engine or graph or production or sharded" > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for v in tools/variants/prev.so ""; do echo "${v:-new}"; SD_LIB_OVERRIDE=$v timeout 120 python tools/draft_bench.py 2>&1 | tail -3; done
for v in tools/variants/prev.so "" tools/variants/prev.so ""; do
  SD_LIB_OVERRIDE=$v timeout 300 python bench.py --no-cpu-baseline --attn-reps 3 2>/dev/null | tail -1 > gpurun_out/ab.json
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('${v:-new}', round(d['ms_per_step'],3), 'ms; draft', round(d['kernels']['draft_attention']['avg_launch_us'],2), 'us', d['clocks']['sm_mhz'])"
done
