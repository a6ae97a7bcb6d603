#!/bin/bash
# verify-kernel skeleton experiments (graph-timed, same box): see SD_TC_EXPERIMENT in attention_tc.cu
export TC_SHAPES="54096,41,32,8;54096,20,32,8;54096,41,8,8"
for v in "" tools/variants/tcexp4.so tools/variants/tcexp5.so tools/variants/tcexp6.so tools/variants/tcexp9.so tools/variants/tcexp8.so; do
  echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 300 python tools/time_tc_cfg.py 2>&1 | tail -3
done
