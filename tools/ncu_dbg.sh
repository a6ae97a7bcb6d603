mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:gemv_tma -c 3 python tools/gemv_bench.py > gpurun_out/ncu_dbg1.log 2>&1; echo "eager rc=$?"; grep -E "ERROR|gemv_tma|duration" gpurun_out/ncu_dbg1.log | head -8
SD_NO_PDL=1 timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_nopdl.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --attn-reps 1 > gpurun_out/ncu_dbg2.log 2>&1; echo "nopdl rc=$?"; grep ERROR gpurun_out/launches_nopdl.csv | head -3; wc -l gpurun_out/launches_nopdl.csv
