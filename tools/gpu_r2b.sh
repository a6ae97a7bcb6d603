# all GPU tests + smoke + a bench line (fused LM head on) and one with it off
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in 1 0 1; do SD_FUSE_LM_HEAD=$f timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_fuse$f.json; python -c "import json; d=json.load(open('gpurun_out/bench_fuse$f.json')); print('fuse=$f', round(d['ms_per_step'],3), 'ms', d['value'], d['gpu_launches'], d['clocks'])"; done
