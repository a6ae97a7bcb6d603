# draft attention shared-memory footprint vs PDL co-residency with the next weight stream
for v in "" tools/variants/dr_nst3.so tools/variants/dr_nst2.so ""; do
  SD_LIB_OVERRIDE=$v timeout 300 python bench.py --no-cpu-baseline --attn-reps 3 2>/dev/null | tail -1 > gpurun_out/drv.json
  python -c "import json; d=json.load(open('gpurun_out/drv.json')); print('$v', round(d['ms_per_step'],3), 'ms; draft attn', round(d['kernels']['draft_attention']['avg_launch_us'],2), 'us')"
done
