#!/bin/bash
# sd_gemm_rows: parity, kernel timing vs cuBLAS, then a same-box step A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm_rows.py -x -q > gpurun_out/rows_tests.log 2>&1; rc=$?; echo "rows tests rc=$rc"; tail -15 gpurun_out/rows_tests.log
[ $rc -ne 0 ] && exit 1
timeout 200 python tools/rows_bench.py
timeout 900 python -m pytest tests/test_gpu_production.py -x -q > gpurun_out/prod_tests.log 2>&1; echo "prod tests rc=$?"; tail -3 gpurun_out/prod_tests.log
for k in "" "wqkv,wo" "" "wqkv,wo"; do
  echo "== SD_ROWS_KEYS=$k"
  SD_ROWS_KEYS=$k timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['value'],1), 'tok/s', d['gpu_launches'], d['clocks']['sm_mhz'])"
done
