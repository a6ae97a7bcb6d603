mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or split_slices" > gpurun_out/gemm2_tests.log 2>&1; tail -1 gpurun_out/gemm2_tests.log
SD_GEMM_REPORT=1 GEMM_MS=101 GEMM_NO_GEMV=1 timeout 300 python tools/gemm_tc_bench.py 2>&1 | grep -v "smem \|sd_gemm M" 
for k in "" "wqkv,wo,w1,w2" "wqkv" "w2" "w1" "wo"; do
  SD_GEMM_KEYS=$k timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_gemm.json
  python -c "import json; d=json.load(open('gpurun_out/bench_gemm.json')); print('keys=$k', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done
