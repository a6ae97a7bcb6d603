#!/bin/bash
export TC_SHAPES="54096,41,32,8;12048,41,32,8;54096,101,32,8"
for v in "" tools/variants/merge4.so tools/variants/merge16.so "" tools/variants/merge16.so; do
  echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 300 python tools/time_tc_cfg.py 2>&1 | tail -3
done
