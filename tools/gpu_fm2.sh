#!/bin/bash
SD_TC_FUSED_MERGE=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "tcgen05 or verify_attention or ctx_dev or rows_dev" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_production.py -x -q -k "tcgen05 or verify_attention or ctx_dev or rows_dev or cfg3" 2>&1 | tail -1
export TC_SHAPES="54096,41,32,8;12048,41,32,8"
for v in 0 1 0; do echo "== SD_TC_FUSED_MERGE=$v"; SD_TC_FUSED_MERGE=$v timeout 120 python tools/time_tc_cfg.py 2>&1 | tail -2; done
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'tok/s', 'attn', round(d['roofline']['avg_launch_us'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
