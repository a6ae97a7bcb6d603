bash tools/gpu_variants.sh | grep -E "==|T=41|T=20"
SD_LIB_OVERRIDE=tools/libsd_trace.so timeout 120 python tools/tc_trace.py 54096 20 8 | tail -11
SD_LIB_OVERRIDE=tools/libsd_trace.so timeout 120 python tools/tc_trace.py 54096 41 8 | tail -11
