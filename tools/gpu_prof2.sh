mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "partial or select or engine or graph or production or sharded or scores" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 120 python tools/refresh_bench.py > gpurun_out/refresh.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:verify_attn_tc -s 3 -c 1 -o gpurun_out/prof_verify_tc -f python tools/time_tc.py > gpurun_out/prof_verify_tc.log 2>&1
SD_NO_PDL=1 timeout 300 python tools/step_profile.py > gpurun_out/step_profile_nopdl.txt 2>&1
tail -3 gpurun_out/pytest_quick.log; cat gpurun_out/refresh.log; head -36 gpurun_out/step_profile_nopdl.txt
