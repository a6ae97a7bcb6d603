#!/bin/bash
export TC_SHAPES="54096,41,32,8;12048,41,32,8"
for v in tools/variants/old_attn.so "" tools/variants/old_attn.so ""; do echo "== ${v:-current}"; SD_LIB_OVERRIDE=$v timeout 120 python tools/time_tc_cfg.py 2>&1 | tail -2; done
