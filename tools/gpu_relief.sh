#!/bin/bash
export TC_SHAPES="54096,41,32,8;12048,41,32,8"
for v in "" tools/variants/relief48.so tools/variants/relief96.so "" tools/variants/relief48.so tools/variants/relief96.so; do echo "== ${v:-default}"; SD_LIB_OVERRIDE=$v timeout 120 python tools/time_tc_cfg.py 2>&1 | tail -2; done
