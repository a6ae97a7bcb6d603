#!/bin/bash
# Round-2 GPU check: production-shape parity first, then the whole GPU suite,
# smoke and a short bench. Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_production.py -q --timeout 600 -rf > gpurun_out/pytest_prod.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_prod.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -rf --deselect tests/test_gpu_production.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -5 gpurun_out/pytest_prod.log; tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/bench.log
