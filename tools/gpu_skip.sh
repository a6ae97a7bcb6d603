#!/bin/bash
# Marginal cost of each kernel family in the real (graph + PDL) cfg3 step:
# bench with that family's launches dropped (SD_DEBUG_SKIP; numbers only, results garbage).
mkdir -p gpurun_out
run() { echo "== $1"; SD_DEBUG_SKIP="$1" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --attn-reps 1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"; }
{
run ""
run "sd_attention:0"
run "sd_attention:1"
run "sd_add_rmsnorm"
run "sd_rope_stage"
run "sd_silu"
run "mm:6144,mm:4096,mm:16384"
run "mm:128256"
run "sd_gemv"
run "sd_sample_rows"
run "sd_draft_topw,sd_draft_tree,sd_accept_commit"
} > gpurun_out/skip.txt 2>&1
cat gpurun_out/skip.txt
