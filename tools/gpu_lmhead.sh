# fused LM head: parity tests + timing vs cuBLAS + sampler (cfg3 shape)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x > gpurun_out/lmhead_tests.log 2>&1; tail -15 gpurun_out/lmhead_tests.log
timeout 300 python tools/lmhead_bench.py 2>&1 | tee gpurun_out/lmhead_bench.log
