#!/bin/bash
# ncu full captures of the sampler, draft top-w and the weight-streaming gemv inside the graph step
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"sample_rows_cluster|draft_topw|gemv|silu_kernel|add_rmsnorm" -s 40 -c 12 \
  -o gpurun_out/prof_small2 -f python tools/step_profile.py --steps 1 > gpurun_out/prof_small2.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_small2.log
