#!/bin/bash
# end-of-round measurement set (1 GPU): full GPU suite, smoke, bench line, launch list, ncu of the verify kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 2 30 > gpurun_out/launch_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 3 -c 1 \
  -o gpurun_out/prof_verify_tc -f python tools/time_tc.py > gpurun_out/prof_verify_tc.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log; grep '^{' gpurun_out/bench.log | cut -c1-300; head -12 gpurun_out/launch_summary.txt
