#!/bin/bash
# Quick GPU iteration: selected tests (pytest -k expr in $1), then a short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -rf ${1:+-k "$1"} > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -4 gpurun_out/pytest_quick.log; tail -2 gpurun_out/bench.log
