# ncu full capture of the fused LM head kernel (cfg3 shape) + the scaled-input sampler
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lmhead_kernel" -s 2 -c 1 \
  -o gpurun_out/ncu_lmhead -f python tools/lmhead_bench.py > gpurun_out/ncu_lmhead.log 2>&1; tail -1 gpurun_out/ncu_lmhead.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sample_rows_cluster" -s 60 -c 1 \
  -o gpurun_out/ncu_sampler_scaled -f python tools/lmhead_bench.py > gpurun_out/ncu_sampler_scaled.log 2>&1; tail -1 gpurun_out/ncu_sampler_scaled.log
