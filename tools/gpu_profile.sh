#!/bin/bash
# Profiling round trip (1 GPU): launch list of the timed bench steps, ncu full capture of the
# verification attention kernel and of the draft decode kernel. Outputs -> gpurun_out/
mkdir -p gpurun_out
NCU=ncu
timeout 900 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/launches_bench.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv 2 30 > gpurun_out/launch_summary.txt 2>&1
cat gpurun_out/launch_summary.txt | head -40
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 3 -c 1 \
  -o gpurun_out/prof_verify_tc -f python tools/time_tc.py > gpurun_out/prof_verify_tc.log 2>&1; echo "prof tc rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 1 \
  -o gpurun_out/prof_decode -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/prof_decode.log 2>&1; echo "prof decode rc=$?"
python tools/time_tc.py > gpurun_out/time_tc.log 2>&1; cat gpurun_out/time_tc.log
