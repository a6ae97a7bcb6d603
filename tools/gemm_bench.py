"""Weight-streaming GEMM rates of the decode step's dense layers under cuBLAS
(torch.mm, bf16 in, fp32 out) for both weight layouts: W [K, N] (x @ W) and
W^T [N, K] (x @ Wt.t()). Weights rotate over copies larger than L2."""
import torch

shapes = {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384), "w2": (16384, 4096), "lm": (4096, 128256)}
dev = "cuda"
for M in (1, 4, 101):
    for name, (K, N) in shapes.items():
        copies = max(2, int(600e6 // (K * N * 2)))
        Ws = [torch.randn(K, N, device=dev).to(torch.bfloat16) for _ in range(copies)]
        Wts = [w.t().contiguous() for w in Ws]
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        res = []
        for lay in ("KN", "NK"):
            def run(i):
                if lay == "KN":
                    return torch.mm(x, Ws[i % copies], out_dtype=torch.float32)
                return torch.mm(x, Wts[i % copies].t(), out_dtype=torch.float32)
            for i in range(5):
                run(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 40
            e0.record()
            for i in range(reps):
                run(i)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            res.append(f"{lay} {us:7.1f} us {K * N * 2 / us / 1e3:6.0f} GB/s")
        print(f"M={M:3d} {name:4s} K={K:5d} N={N:6d}: " + " | ".join(res), flush=True)
        del Ws, Wts
