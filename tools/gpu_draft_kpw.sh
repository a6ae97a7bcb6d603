# draft attention keys-per-warp sweep (no-PDL warm step profile)
for k in 16 32 24; do
  touch paper_2502_18890_b200/csrc/attention.cu
  NVCC_EXTRA="-DSD_DR_KPW=$k" timeout 200 python -m paper_2502_18890_b200.build_lib > /dev/null 2>&1
  echo "KPW $k"; SD_NO_PDL=1 timeout 300 python tools/step_profile.py 2>&1 | grep "^step\|draft_attn"
done
