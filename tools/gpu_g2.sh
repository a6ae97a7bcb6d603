bash tools/gpu_variants.sh | grep -E "==|T=41|T=20"
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "tcgen05 or production" 2>&1 | tail -2
