#!/bin/bash
export TC_SHAPES="54096,41,32,8;12048,41,32,8;4096,41,32,8"
for v in "" tools/variants/nomerge.so "" tools/variants/nomerge.so; do
  echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 300 python tools/time_tc_cfg.py 2>&1 | tail -3
done
