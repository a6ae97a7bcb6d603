#!/bin/bash
for u in 8 16; do for c in 2 4 8; do
  touch paper_2502_18890_b200/csrc/gemv.cu
  NVCC_EXTRA="-DSD_GEMV_UNROLL=$u -DSD_GEMV_CTAS_PER_SM=$c" timeout 120 python -m paper_2502_18890_b200.build_lib > /dev/null 2>&1
  echo "unroll $u ctas/sm $c"; timeout 120 python tools/gemm_tc_bench.py 2>&1 | grep gemv | sed 's/cublas.*| //'
done; done
