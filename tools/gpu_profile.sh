#!/bin/bash
# Profiling round trip (1 GPU): bench line, warm step profile, launch list of the timed steps, ncu full
# captures of the verify attention, draft attention, gemv and the cluster sampler. Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 300 python tools/step_profile.py > gpurun_out/step_profile.txt 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/launches_bench.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv 2 30 > gpurun_out/launch_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 3 -c 1 \
  -o gpurun_out/prof_verify_tc -f python tools/time_tc.py > gpurun_out/prof_verify_tc.log 2>&1; echo "prof tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"draft_attn|gemv_tma|sample_rows_cluster|merge128" -s 200 -c 6 \
  -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/prof_chain.log 2>&1; echo "prof chain rc=$?"
