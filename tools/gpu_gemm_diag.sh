# verify-forward GEMM diagnosis: sd_gemm vs cuBLAS per shape, then ncu of each on wqkv / wo at M=101
python -c "import paper_2502_18890_b200._lib as L; L.load()" || exit 1
GEMM_MS=41,101 GEMM_NO_GEMV=1 timeout 300 python tools/gemm_tc_bench.py 2>&1 | tee gpurun_out/gemm_diag.log
for s in qkv wo; do
  for impl in sd_gemm cublas; do
    GEMM_MS=101 GEMM_NO_GEMV=1 GEMM_SHAPES=$s GEMM_IMPLS=$impl timeout 600 ncu --set full --clock-control none -k regex:"gemm_stream|nvjet" -s 10 -c 1 \
      -o gpurun_out/ncu_gemm_${s}_${impl} -f python tools/gemm_tc_bench.py > gpurun_out/ncu_gemm_${s}_${impl}.log 2>&1
    tail -2 gpurun_out/ncu_gemm_${s}_${impl}.log
  done
done
