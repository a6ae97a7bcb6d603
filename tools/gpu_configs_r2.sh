#!/bin/bash
# bench lines for every BASELINE config on one B200 (cfg3 is the default bench line)
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"; grep '^{' gpurun_out/bench_$c.log | tail -1 >> gpurun_out/bench_configs.jsonl
done
