"""Time (and, under ncu, capture) one fused partial-cache refresh at cfg3
shapes: sd_partial_refresh over L layers, ctx rows, budget 4096, sink 32.

    python tools/refresh_bench.py [ctx] [L]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_18890_b200 import FullCache  # noqa: E402
from paper_2502_18890_b200.kvcache import PartialCache  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 54096
Ln = int(sys.argv[2]) if len(sys.argv) > 2 else 32
Hk, H, dh, S, B = 8, 32, 128, 32, 4096
F = FullCache(Ln, Hk, dh, capacity=ctx + 8, dtype=torch.bfloat16)
F.k_raw.normal_()
F.v.normal_()
q = torch.randn((Ln, H, dh), device="cuda")
p = PartialCache(S, B, Ln, Hk, dh, torch.bfloat16, "cuda")
for _ in range(2):
    p.refresh_from(F, ctx, q_sum=q, num_heads=H)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    p.refresh_from(F, ctx, q_sum=q, num_heads=H)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
n = ctx - S
alg = Ln * (n * Hk * dh * 2 + 2 * n * 4 + 2 * (B - S) * Hk * dh * 2 * 2)
print(f"refresh ctx={ctx} L={Ln}: {us:.1f} us, {alg / us / 1e3:.0f} GB/s algorithmic")
