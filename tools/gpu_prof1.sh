mkdir -p gpurun_out
SD_LIB_OVERRIDE=tools/libsd_trace.so timeout 120 python tools/tc_trace.py 54096 41 8 > gpurun_out/trace.log 2>&1
timeout 120 python tools/refresh_bench.py > gpurun_out/refresh.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/prof_refresh -f python tools/refresh_bench.py 54096 32 > gpurun_out/prof_refresh.log 2>&1
timeout 300 python tools/step_profile.py > gpurun_out/step_profile.txt 2>&1
cat gpurun_out/trace.log gpurun_out/refresh.log; head -40 gpurun_out/step_profile.txt
