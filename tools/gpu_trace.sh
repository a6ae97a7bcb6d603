mkdir -p gpurun_out
SD_TC_TRACE=1 NVCC_EXTRA="$TC_EXTRA" python -m paper_2502_18890_b200.build_lib --force > gpurun_out/trace_build.log 2>&1
for a in ${TC_SHAPES:-"54096 41"}; do timeout 60 python tools/tc_trace.py $a 8 > gpurun_out/trace.log 2>&1; cat gpurun_out/trace.log; done
