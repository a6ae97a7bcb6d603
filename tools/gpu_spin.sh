#!/bin/bash
export TC_SHAPES="54096,41,32,8;54096,20,32,8;12048,41,32,8"
for v in "" tools/variants/tcspin.so "" tools/variants/tcspin.so tools/variants/tcexp4.so tools/variants/tcexp4spin.so; do
  echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 300 python tools/time_tc_cfg.py 2>&1 | tail -3
done
