"""Verify-forward projections (M = 101) through torch.mm: default cuBLAS heuristic
vs PyTorch TunableOp (benchmarks the cuBLAS / cuBLASLt algorithms per shape).
Weights rotate over copies larger than L2.

    python tools/tunable_bench.py            # heuristic
    PYTORCH_TUNABLEOP_ENABLED=1 PYTORCH_TUNABLEOP_VERBOSE=0 python tools/tunable_bench.py
"""
import os

import torch

shapes = {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384), "w2": (16384, 4096)}
M = 101
dev = "cuda"


def timeit(fn, reps=5, inner=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / inner * 1e3)
    return best


print("tunable:", os.environ.get("PYTORCH_TUNABLEOP_ENABLED", "0"), flush=True)
x = (torch.randn(M, 16384, device=dev) * 0.1).to(torch.bfloat16)
for name, (K, N) in shapes.items():
    copies = max(2, int(600e6 // (K * N * 2)))
    Ws = [torch.empty(K, N, device=dev, dtype=torch.bfloat16).normal_(0, 0.02) for _ in range(copies)]
    xk = x[:, :K].contiguous()
    out = []
    for label, kw in (("f32out", {"out_dtype": torch.float32}), ("bf16out", {})):
        it = iter(range(1 << 30))
        try:
            us = timeit(lambda: torch.mm(xk, Ws[next(it) % copies], **kw))
            out.append(f"{label} {us:5.1f} us {K * N * 2 / us / 1e3:5.0f} GB/s")
        except Exception as e:  # out_dtype may not be tunable
            out.append(f"{label} error {str(e)[:60]}")
    print(f"{name:4s}: " + " | ".join(out), flush=True)
    del Ws
