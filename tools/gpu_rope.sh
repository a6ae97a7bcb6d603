#!/bin/bash
SD_ROPE_SPREAD=1 timeout 600 python -m pytest tests/test_gpu_production.py -x -q 2>&1 | tail -1
for v in 0 1 0 1 0 1; do
  echo "== SD_ROPE_SPREAD=$v"
  SD_ROPE_SPREAD=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'tok/s', d['clocks']['sm_mhz'])"
done
