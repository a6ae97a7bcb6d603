"""Verify-forward projections (M = 101 padded tree rows) through cuBLAS: one
torch.mm vs a K-split batched GEMM whose [S, M, N] fp32 slices the consumers
(sd_rope_stage / sd_add_rmsnorm) sum in order. Weights rotate over copies
larger than L2."""
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


x = (torch.randn(M, 16384, device=dev) * 0.1).to(torch.bfloat16)
for name, (K, N) in shapes.items():
    copies = max(2, int(600e6 // (K * N * 2)))
    Ws = [torch.empty(K, N, device=dev, dtype=torch.bfloat16).normal_(0, 0.02) for _ in range(copies)]
    xk = x[:, :K].contiguous()
    ref = torch.mm(xk, Ws[0], out_dtype=torch.float32)
    out = []
    for S in (1, 2, 3, 4, 6, 8):
        if K % S:
            continue
        it = iter(range(1 << 30))
        if S == 1:
            fn = lambda: torch.mm(xk, Ws[next(it) % copies], out_dtype=torch.float32)
        else:
            x3 = xk.view(M, S, K // S).transpose(0, 1)
            fn = lambda: torch.bmm(x3, Ws[next(it) % copies].view(S, K // S, N), out_dtype=torch.float32)
            y = torch.bmm(x3, Ws[0].view(S, K // S, N), out_dtype=torch.float32)
            acc = y[0].clone()
            for s in range(1, S):
                acc += y[s]
            err = (acc - ref).abs().max().item()
            assert err < 1e-2, (name, S, err)
        us = timeit(fn)
        out.append(f"S={S} {us:5.1f} us {K * N * 2 / us / 1e3:5.0f} GB/s")
    print(f"{name:4s}: " + " | ".join(out), flush=True)
    del Ws
