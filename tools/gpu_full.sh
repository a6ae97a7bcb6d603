# full GPU check: all -m gpu tests, smoke, sanitizer passes; logs -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_sanitize.sh
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
