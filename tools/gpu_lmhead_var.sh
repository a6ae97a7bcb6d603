for V in 128256; do LMH_TIME=1 LMH_V=$V SD_LIB_OVERRIDE=tools/variants/lh_time.so timeout 120 python tools/lmhead_bench.py 2>&1 | grep "min_p.*only\|cta"; done
