#!/bin/bash
# Debug: time the tcgen05 verify kernel with pipeline pieces disabled (SD_TC_EXPERIMENT builds).
for e in "-DSD_TC_EXPERIMENT=6" "-DSD_TC_EXPERIMENT=4" "-DSD_TC_EXPERIMENT=1"; do
  NVCC_EXTRA="$e" timeout 200 python -m paper_2502_18890_b200.build_lib --force > /dev/null 2>&1
  echo "experiment $e"; timeout 60 python tools/time_tc.py 2>&1 | head -4
done
