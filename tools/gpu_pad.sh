mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pad_tests.log 2>&1; tail -1 gpurun_out/pad_tests.log
for f in 0 1 0 1 0 1; do
  SD_GEMM_PAD=$f timeout 300 python bench.py --no-cpu-baseline --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/pad.json
  python -c "import json; d=json.load(open('gpurun_out/pad.json')); print('pad=$f', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done
