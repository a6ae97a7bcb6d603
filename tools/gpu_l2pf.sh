# L2 weight prefetch during the verify attention: step time A/B (bench.py, cfg3 ctx 54096)
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms', round(d['roofline']['avg_launch_us'],1), 'us attn', d['clocks']['sm_mhz'])"; }
{
run SD_L2_PREFETCH=
run SD_LIB_OVERRIDE=tools/variants/nohint.so SD_L2_PREFETCH=
run SD_L2_PREFETCH=wo
run SD_L2_PREFETCH=wo SD_L2_PF_LAST=0
run SD_LIB_OVERRIDE=tools/variants/nohint.so SD_L2_PREFETCH=wo
run SD_L2_PREFETCH=wo,wqkv+
run SD_L2_PREFETCH=wo,w1
run SD_L2_PREFETCH=
} > gpurun_out/l2pf.log 2>&1
cat gpurun_out/l2pf.log
