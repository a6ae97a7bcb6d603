#!/bin/bash
# tcgen05 verify kernel: parity tests + timing (1 GPU)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "tcgen05 or verify_attention" > gpurun_out/tc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tc_tests.log
tail -3 gpurun_out/tc_tests.log
timeout 120 python tools/time_tc.py > gpurun_out/time_tc.log 2>&1; cat gpurun_out/time_tc.log
