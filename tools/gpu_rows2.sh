#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_gemm_rows.py -x -q 2>&1 | tail -2
timeout 200 python tools/rows_bench.py
for k in "" "wqkv,wo" "" "wqkv,wo"; do
  echo "== SD_ROWS_KEYS=$k"
  SD_ROWS_KEYS=$k timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'tok/s', d['gpu_launches'], d['clocks']['sm_mhz'])"
done
for k in "" "wqkv,wo"; do echo "== profile SD_ROWS_KEYS=$k"; SD_NO_PDL=1 SD_ROWS_KEYS=$k timeout 300 python tools/step_profile.py 2>&1 | grep -E "gemm_rows|nvjet|rmsnorm|rope_stage|^step"; done
