# step-graph edge relaxation (cuBLAS -> our kernels at launch completion): correctness + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_production.py -q -x --timeout 600 > gpurun_out/relax_tests.log 2>&1; tail -2 gpurun_out/relax_tests.log
python - <<'PY'
import bench, sys
PY
for r in 1 0 1 0; do
  SD_RELAX_EDGES=$r timeout 300 python bench.py --no-cpu-baseline --attn-reps 1 2>/dev/null | tail -1 > gpurun_out/relax.json
  python -c "import json; d=json.load(open('gpurun_out/relax.json')); print('relax=$r', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done
