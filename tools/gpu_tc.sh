#!/bin/bash
# tcgen05 verify kernel: parity tests (repeated) + timing (1 GPU)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "tcgen05 or verify_attention or ctx_dev" --count 1 > gpurun_out/tc_tests.log 2>&1 || \
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "tcgen05 or verify_attention or ctx_dev" > gpurun_out/tc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tc_tests.log
tail -3 gpurun_out/tc_tests.log
for i in 1 2 3; do timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "tcgen05" 2>&1 | tail -1; done
timeout 120 python tools/time_tc.py > gpurun_out/time_tc.log 2>&1; cat gpurun_out/time_tc.log
