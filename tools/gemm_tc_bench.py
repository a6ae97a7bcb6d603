"""sd_gemm (tcgen05 weight-streaming) vs cuBLAS on the decode shapes; weights
rotate over copies larger than L2."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import _lib as L  # noqa: E402

shapes = {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384), "w2": (16384, 4096)}
if os.environ.get("GEMM_SHAPES"):
    shapes = {k: v for k, v in shapes.items() if k in os.environ["GEMM_SHAPES"].split(",")}
IMPLS = tuple(os.environ.get("GEMM_IMPLS", "cublas,sd_gemm").split(","))
dev = "cuda"
for M in [int(m) for m in os.environ.get("GEMM_MS", "1,101").split(",")]:
    for name, (K, N) in shapes.items():
        copies = max(2, int(600e6 // (K * N * 2)))
        Ws = [(torch.randn(K, N, device=dev) * 0.02).to(torch.bfloat16) for _ in range(copies)]
        tms, wts = [], []
        for w in Ws:
            wt = torch.empty((N // 128, 2, K, 64), dtype=torch.bfloat16, device=dev)
            L.call("sd_tile_weight", L.ptr(w), K, N, L.ptr(wt), L.stream())
            tm = ctypes.create_string_buffer(128)
            L.call("sd_make_weight_tmap", L.ptr(wt), K, N, tm)
            tms.append(tm)
            wts.append(wt)

        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        y = torch.empty(12, M, N, device=dev)
        epi = 1 if name == "w1" else 0
        ws = torch.zeros(max(256, L.load().sd_gemm_workspace_bytes(M, N, K)), dtype=torch.uint8, device=dev)
        out = []
        for impl in IMPLS:
            def run(i):
                if impl == "cublas":
                    torch.mm(x, Ws[i % copies], out_dtype=torch.float32)
                else:
                    L.call("sd_gemm", L.ptr(x), M, K, tms[i % copies], N, epi, L.ptr(y), N, L.ptr(ws), ws.numel(), L.stream())
            for i in range(5):
                run(i)
            torch.cuda.synchronize()
            best = 1e9
            for rep in range(5):  # best of 5 batches of 20 (the pool's boxes are noisy)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(20):
                    run(i)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
            us = best
            out.append(f"{impl} {us:6.1f} us {K * N * 2 / us / 1e3:5.0f} GB/s")
        print(f"M={M:3d} {name:4s}: " + " | ".join(out), flush=True)

# single-row weight streaming (sd_gemv) vs cuBLAS
if os.environ.get("GEMM_NO_GEMV"):
    sys.exit(0)
for name, (K, N) in list(shapes.items()) + [("head", (4096, 4096))]:
    copies = max(2, int(600e6 // (K * N * 2)))
    Ws = [(torch.randn(K, N, device=dev) * 0.02).to(torch.bfloat16) for _ in range(copies)]
    ws = torch.zeros(max(256, L.load().sd_gemv_workspace_bytes(K, N)), dtype=torch.uint8, device=dev)
    x = torch.randn(1, K, device=dev).to(torch.bfloat16)
    y = torch.empty(1, N, device=dev)
    out = []
    for impl in ("cublas", "sd_gemv"):
        def run(i):
            if impl == "cublas":
                torch.mm(x, Ws[i % copies], out_dtype=torch.float32)
            else:
                L.call("sd_gemv", L.ptr(x), K, L.ptr(Ws[i % copies]), N, 0, L.ptr(y), L.ptr(ws), ws.numel(), L.stream())
        for i in range(5):
            run(i)
        torch.cuda.synchronize()
        best = 1e9
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(20):
                run(i)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
        out.append(f"{impl} {best:6.1f} us {K * N * 2 / best / 1e3:5.0f} GB/s")
    print(f"M=  1 {name:4s} (gemv): " + " | ".join(out), flush=True)
