bash tools/gpu_variants.sh
SD_NO_PDL=1 timeout 300 python tools/step_profile.py 2>&1 | grep -E "step|partial_step|verify_attn"
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "partial or select or engine" 2>&1 | tail -2
