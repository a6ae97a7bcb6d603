# verify-forward projections: cuBLAS vs sd_gemm (PDL) per projection, whole-step times
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gemm" > gpurun_out/gemm_tests.log 2>&1; tail -2 gpurun_out/gemm_tests.log
for k in "" "wqkv" "wo" "wqkv,wo" "wqkv,wo,w2" "wqkv,wo,w1,w2"; do
  echo "== SD_GEMM_KEYS=$k"; SD_GEMM_KEYS=$k timeout 300 python tools/step_profile.py 2>&1 | grep "^step\|gemm_stream\|nvjet"
done
