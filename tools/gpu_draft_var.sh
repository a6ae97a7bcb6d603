for v in tools/variants/d_*.so; do echo "== $v"; SD_LIB_OVERRIDE=$v timeout 120 python tools/draft_bench.py 2>&1 | tail -2; done
