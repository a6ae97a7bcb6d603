# Round-2 final measurement set (1 GPU): GPU tests + smoke, bench line (with the CPU baseline),
# n-gram stress line, ncu launch list of the timed steps, ncu full capture of the fused LM head,
# the 100K-token generation. Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --ngram-stress > gpurun_out/bench_stress.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 2 30 > gpurun_out/launch_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lmhead_kernel" -s 2 -c 1 \
  -o gpurun_out/prof_lmhead -f python tools/lmhead_bench.py > gpurun_out/prof_lmhead.log 2>&1
timeout 900 python tools/run_100k.py --out gpurun_out/run_100k.json > gpurun_out/run_100k.log 2>&1; echo "run_100k rc=$?" >> gpurun_out/run_100k.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-300; tail -3 gpurun_out/run_100k.log
