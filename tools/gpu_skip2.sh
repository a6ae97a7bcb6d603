# marginal cost of each launch family inside the real (graph + PDL) cfg3 step: drop it, re-time
mkdir -p gpurun_out
for k in "" "sd_rope_stage:1" "sd_rope_stage:101" "sd_add_rmsnorm:101" "sd_add_rmsnorm:1" "sd_silu" "sd_attention:1" "sd_attention:0" "mm:6144" "mm:4096" "mm:16384" "mm:128256" "sd_sample_rows" "sd_lmhead_sample_stats" "sd_draft_topw" ""; do
  SD_DEBUG_SKIP=$k timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/skip.json
  python -c "import json; d=json.load(open('gpurun_out/skip.json')); print('skip=$k', round(d['ms_per_step'],3), 'ms')" 2>/dev/null || echo "skip=$k failed"
done
