# Round-2 profile set (1 GPU): bench line, bench --ngram-stress line, ncu launch list of the timed
# steps, ncu --set full of the verify attention (T=41 and T=101), the refresh and the draft attention,
# warm per-kernel step profile without PDL. Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --ngram-stress > gpurun_out/bench_stress.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 \
  > gpurun_out/launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 2 30 > gpurun_out/launch_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 3 -c 1 \
  -o gpurun_out/prof_verify_tc -f python tools/time_tc.py > gpurun_out/prof_verify_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 46 -c 1 \
  -o gpurun_out/prof_verify_tc_t101 -f python tools/time_tc.py > gpurun_out/prof_verify_tc_t101.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 \
  -o gpurun_out/prof_refresh -f python tools/refresh_bench.py 54096 32 > gpurun_out/prof_refresh.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:draft_mma -s 40 -c 1 \
  -o gpurun_out/prof_draft -f python tools/draft_bench.py > gpurun_out/prof_draft.log 2>&1
SD_NO_PDL=1 timeout 300 python tools/step_profile.py > gpurun_out/step_profile_nopdl.txt 2>&1
tail -1 gpurun_out/bench.log | cut -c1-400; head -30 gpurun_out/launch_summary.txt
