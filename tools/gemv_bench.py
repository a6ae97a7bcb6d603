"""sd_gemv on the draft-forward shapes: each shape alone (weights rotating over
copies larger than L2) and the whole 32-layer chain qkv -> wo -> w1 -> w2 as
one stream of PDL launches (11 GB of distinct weights, as in the draft step)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import _lib as L  # noqa: E402

shapes = {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384), "w2": (16384, 4096)}
dev = "cuda"
x = (torch.randn(1, 16384, device=dev) * 0.1).to(torch.bfloat16)
y = torch.empty(16384, device=dev)
ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)


def gemv(w, K, N, epi=0):
    L.call("sd_gemv", L.ptr(x), K, L.ptr(w), N, epi, L.ptr(y), L.ptr(ws), ws.numel(), L.stream())


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


tot = 0
for name, (K, N) in shapes.items():
    copies = max(2, int(600e6 // (K * N * 2)))
    Ws = [torch.empty(K, N, device=dev, dtype=torch.bfloat16).normal_(0, 0.02) for _ in range(copies)]
    it = iter(range(1 << 30))
    us = timeit(lambda: gemv(Ws[next(it) % copies], K, N))
    tot += K * N * 2
    print(f"{name:4s} {us:6.1f} us {K * N * 2 / us / 1e3:5.0f} GB/s", flush=True)
    del Ws

layers = 32
Wl = [[torch.empty(K, N, device=dev, dtype=torch.bfloat16).normal_(0, 0.02) for (K, N) in shapes.values()]
      for _ in range(layers)]


def chain():
    for l in range(layers):
        for (K, N), w in zip(shapes.values(), Wl[l]):
            gemv(w, K, N)


us = timeit(chain, reps=3, inner=3)
print(f"chain {layers}x4: {us:8.1f} us  {layers * tot / us / 1e3:5.0f} GB/s  ({us / layers:5.1f} us/layer)", flush=True)
