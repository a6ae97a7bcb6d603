"""sd_gemm_rows vs cuBLAS on the verify projections (T=101 padded, 41 live rows),
32 distinct weight copies per shape (> L2), graph-replayed back to back."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import _lib as L  # noqa: E402

L.load()


def gtime(fn, reps=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
    return best * 1e3


T, live = 101, int(os.environ.get("LIVE", "41"))
rows = torch.tensor([live], dtype=torch.int32, device="cuda")
for name, (K, N) in {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384), "w2": (16384, 4096)}.items():
    n = 32 if K * N * 2 * 32 > 200e6 else 64
    Ws = [(torch.randn(K, N, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(n)]
    x = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    S = L.load().sd_gemm_rows_splits(K, N)
    y = torch.empty((S, T, N), dtype=torch.float32, device="cuda")

    def cub():
        for w in Ws:
            torch.mm(x, w, out_dtype=torch.float32)

    def rows_k():
        for w in Ws:
            L.call("sd_gemm_rows", L.ptr(x), T, K, L.ptr(w), N, L.ptr(rows), L.ptr(y), L.stream())
    tc, tr = gtime(cub) / n, gtime(rows_k) / n
    mb = K * N * 2 / 1e6
    print(f"{name} K={K} N={N} S={S}: cuBLAS {tc:.1f} us ({mb / tc:.2f} TB/s)  rows {tr:.1f} us ({mb / tr:.2f} TB/s)")
