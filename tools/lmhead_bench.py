"""Verification LM head + sampler at the cfg3 shape (T=101 padded rows, 41 live,
V=128256, d=4096): cuBLAS fp32-out GEMM + engine sampler vs the fused tcgen05
LM head (sd_lmhead_sample_stats) + the sampler's scaled-input path."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import _lib as Lb  # noqa: E402
import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location("tglh", "tests/test_gpu_lmhead.py")
_m = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_m)
_args, _tree_and_window = _m._args, _m._tree_and_window

import os  # noqa: E402

V, K, T = int(os.environ.get("LMH_V", 128256)), 4096, int(os.environ.get("LMH_T", 101))
g = np.random.default_rng(0)
st, dw, rec, W = _tree_and_window(Lb, V, g)
E = (torch.randn((V, K), device="cuda") * (3.0 / K ** 0.5)).to(torch.bfloat16)
x = torch.randn((T, K), device="cuda").to(torch.bfloat16)
tm = ctypes.create_string_buffer(128)
Et = torch.empty(Lb.load().sd_lmhead_tiled_bytes(V, K), dtype=torch.uint8, device="cuda")
Lb.call("sd_tile_lmhead", Lb.ptr(E), V, K, Lb.ptr(Et), Lb.stream())
Lb.call("sd_make_lmhead_tmap", Lb.ptr(Et), V, K, tm)
tiles = Lb.load().sd_lmhead_tiles(V)
s = torch.empty((T, V), device="cuda")
stats = torch.empty((T, tiles, 2), dtype=torch.float64, device="cuda")
y = torch.empty((T,), dtype=torch.int32, device="cuda")
for trunc, code, val in (("min_p", Lb.TRUNC_MIN_P, 0.1), ("top_p", Lb.TRUNC_TOP_P, 0.9)):
    a = _args(Lb, T, V, st, dw, rec, W, code, val, 0)
    a.token_out = Lb.ptr(y)
    a3 = _args(Lb, T, V, st, dw, rec, W, code, val, 0)
    a3.token_out = Lb.ptr(y)

    def unfused():
        raw = torch.mm(x, E.t(), out_dtype=torch.float32)
        Lb.call("sd_sample_rows", Lb.ptr(raw), a, Lb.stream())

    def gemm_only():
        torch.mm(x, E.t(), out_dtype=torch.float32)

    def fused():
        a3.in_kind, a3.stats, a3.stats_tiles = Lb.IN_LOGITS_F32, None, 0
        Lb.call("sd_lmhead_sample_stats", Lb.ptr(x), T, K, tm, V, a3, Lb.ptr(s), Lb.ptr(stats), Lb.stream())
        a3.in_kind, a3.stats, a3.stats_tiles = Lb.IN_SCALED_F32, Lb.ptr(stats), tiles
        Lb.call("sd_sample_rows", Lb.ptr(s), a3, Lb.stream())

    def lmhead_only():
        a3.in_kind, a3.stats, a3.stats_tiles = Lb.IN_LOGITS_F32, None, 0
        Lb.call("sd_lmhead_sample_stats", Lb.ptr(x), T, K, tm, V, a3, Lb.ptr(s), Lb.ptr(stats), Lb.stream())

    for name, fn in (("cublas+sampler", unfused), ("cublas gemm", gemm_only), ("fused", fused),
                     ("fused lmhead only", lmhead_only)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 10 * 1e3)
        print(f"{trunc:6s} {name:18s} {best:7.1f} us  ({V * K * 2 / best / 1e3:5.0f} GB/s embed stream)", flush=True)

if os.environ.get("LMH_TIME"):
    lmhead_only()
    torch.cuda.synchronize()
    st = stats.view(-1)[: 148 * 16].view(148, 16).cpu().numpy()
    ends = [(st[g, 2 + int(st[g, 1]) - 1], g) for g in range(148)]
    ends.sort()
    for e, g in ends[-3:] + ends[:2]:
        n = int(st[g, 1])
        print("cta %3d tiles %d bloom %d: " % (g, st[g, 0], st[g, 14]) + " ".join("%.1f" % (x / 1e3) for x in st[g, 2:2 + n]))
