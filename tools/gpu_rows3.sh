#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_gemm_rows.py tests/test_gpu_production.py -x -q 2>&1 | tail -2
for cap in 9 6 4 3 2; do echo "== cap $cap"; SD_ROWS_MAX_SPLITS=$cap timeout 200 python tools/rows_bench.py | head -2; done
for cfg in ":" "wqkv,wo:" "wqkv,wo:4" "wqkv,wo:3" ":" "wqkv,wo:" "wqkv,wo:4" "wqkv,wo:2"; do
  k=${cfg%%:*}; cap=${cfg##*:}
  echo "== SD_ROWS_KEYS=$k cap=$cap"
  SD_ROWS_MAX_SPLITS=$cap SD_ROWS_KEYS=$k timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'tok/s', d['clocks']['sm_mhz'])"
done
