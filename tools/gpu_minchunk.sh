#!/bin/bash
# verify attention min-chunk sweep (same box): default 256 vs variants
for v in "" tools/variants/minchunk64.so tools/variants/minchunk128.so tools/variants/minchunk192.so; do
  echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 300 python tools/time_tc_cfg.py 2>&1 | tail -6
done
for v in ""; do
  echo "== draft ${v:-default}"
  SD_LIB_OVERRIDE=$v timeout 120 python tools/draft_bench.py --H 12 --Hk 2 --slots 2056 --L 28 2>&1 | tail -1
  SD_LIB_OVERRIDE=$v timeout 120 python tools/draft_bench.py 2>&1 | tail -1
done
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 bench verify', d['roofline']['avg_launch_us'], d['roofline']['frac'])"
