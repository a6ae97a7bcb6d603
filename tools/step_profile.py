"""Warm per-kernel device times of the decode step (torch.profiler / CUPTI,
graph-replayed kernels included). Unlike an ncu launch list, caches are warm
and kernels overlap exactly as in the bench.

    python tools/step_profile.py [--config cfg3] [--ctx 54096] [--steps 5] [--eager]
"""
import argparse
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_18890_b200 as sd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--ctx", type=int, default=None)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--eager", action="store_true")
args = ap.parse_args()
c = bench.CONFIGS[args.config]
ctx = args.ctx or c["prefix"] + c["gen"] // 2
mcfg = sd.ModelConfig(vocab_size=c["V"], num_layers=c["L"], hidden_dim=c["d"], num_heads=c["H"], num_kv_heads=c["Hk"],
                      gamma=3, max_positions=c["prefix"] + c["gen"] + 256, init_seed=0)
model = sd.TinyTransformer(mcfg, dtype=torch.bfloat16, init="device")

ecfg = sd.EngineConfig(target_length=c["gen"], sink_size=c["S"], budget=c["B"], tree=sd.TreeConfig((1, 3, 3, 3)), k=20,
                       sampler=sd.SamplerConfig(theta=c["theta"], window=1024, truncation=sd.Truncation(*c["trunc"])))
sess = sd.Session(model, sd.rng.random_prompt(c["prefix"], c["V"]), ecfg, capacity=c["prefix"] + c["gen"] + 512,
                  graph=not args.eager)
sess.set_synthetic_context(ctx)
for _ in range(4):
    sess.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    sess.step()
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1) / args.steps
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        sess.step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v for _, v in agg.values())
print(f"step {step_ms:.3f} ms (events, unprofiled); kernel time {tot / args.steps / 1e3:.3f} ms/step; "
      f"{sum(n for n, _ in agg.values()) / args.steps:.0f} kernels/step")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v / tot * 100:6.2f}%  {v / args.steps:9.1f} us/step  {n / args.steps:5.0f}/step  {v / n:8.2f} us  {k}")
