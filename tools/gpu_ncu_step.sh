# ncu full captures of the step's smaller kernels, taken inside the timed graph replays of bench.py
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:"${NCU_K:-sample_rows_cluster|draft_attn|gemv_tma|merge128|draft_topw|add_rmsnorm|rope_stage}" -c ${NCU_C:-14} \
  -o gpurun_out/prof_step -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/prof_step.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/prof_step.log
