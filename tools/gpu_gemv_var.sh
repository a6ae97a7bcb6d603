#!/bin/bash
# gemv variants on the draft shapes + the 32-layer chain, then whole-step times
# args per variant: impl pipe unroll minb tr ns cps
mkdir -p gpurun_out
run() {
  touch paper_2502_18890_b200/csrc/gemv.cu
  NVCC_EXTRA="-DSD_GEMV_PIPE=$2 -DSD_GEMV_UNROLL=$3 -DSD_GEMV_MINB=$4 -DSD_GEMV_TR=$5 -DSD_GEMV_NS=$6 -DSD_GEMV_TMA_CPS=$7" \
    timeout 200 python -m paper_2502_18890_b200.build_lib > /dev/null 2>&1
  echo "== $*"; SD_GEMV_IMPL=$1 timeout 200 python tools/gemv_bench.py 2>&1 | tail -5
  if [ -n "$STEP" ]; then SD_GEMV_IMPL=$1 timeout 300 python tools/step_profile.py 2>&1 | grep "^step\|gemv"; fi
}
STEP=1 run tma 0 8 4 32 8 1
STEP=1 run tma 0 8 4 32 10 1
STEP=1 run tma 0 8 4 32 12 1
STEP=1 run tma 0 8 4 64 6 1
