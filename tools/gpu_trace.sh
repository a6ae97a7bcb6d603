mkdir -p gpurun_out
SD_TC_TRACE=1 NVCC_EXTRA="$TC_EXTRA" python -m paper_2502_18890_b200.build_lib --force > gpurun_out/trace_build.log 2>&1
timeout 60 python tools/tc_trace.py ${TC_CTX:-54096} ${TC_T:-41} 8 > gpurun_out/trace.log 2>&1; cat gpurun_out/trace.log
