#!/bin/bash
# One ncu --set full capture of the cluster verify kernel at cfg3 T=41 (verify_bench's first timed shape)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:verify_mc -s 6 -c 1 -o gpurun_out/verify_mc -f python tools/verify_bench.py > gpurun_out/ncu_verify_mc.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_verify_mc.log
tail -3 gpurun_out/ncu_verify_mc.log
