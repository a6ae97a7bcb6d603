# tcgen05 verify-attention correctness + timing (one GPU call)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "tcgen05 or production or verify" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
timeout 120 python tools/time_tc.py > gpurun_out/time_tc.log 2>&1
tail -3 gpurun_out/pytest_tc.log; cat gpurun_out/time_tc.log
