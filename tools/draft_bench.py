"""Draft attention alone at cfg-shaped partial caches: the tensor-core kernel
(TMA slot descriptors) vs the CUDA-core kernel, CUDA-graph timed, 32 layers
back to back (each layer's slots a distinct buffer). Prints GB/s and the
fraction of the measured HBM peak.

    python tools/draft_bench.py [--Hk 8 --H 32 --slots 4104 --L 32]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_18890_b200 import _lib as L  # noqa: E402


def graph_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--Hk", type=int, default=8)
    ap.add_argument("--slots", type=int, default=4104)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = L.load()
    dh, H, Hk, Ln, cap = 128, a.H, a.Hk, a.L, a.slots
    dev = "cuda"
    pk = torch.randn((Ln, Hk, cap, dh), device=dev).to(torch.bfloat16)
    pv = torch.randn_like(pk)
    rank = torch.stack([torch.randperm(cap, device=dev, dtype=torch.int32) for _ in range(Ln)])
    rank[:, ::97] = -1
    maxpos = cap + 16
    inv = 10000.0 ** (-torch.arange(0, dh, 2, dtype=torch.float64) / dh)
    ang = torch.arange(maxpos, dtype=torch.float64)[:, None] * inv[None, :]
    cos_t, sin_t = ang.cos().float().to(dev), ang.sin().float().to(dev)
    q = (torch.randn((1, H, dh), device=dev) * 0.1).to(torch.bfloat16)
    kt = torch.randn((Hk, dh), device=dev).to(torch.bfloat16)
    vt = torch.randn_like(kt)
    out = torch.empty((1, H * dh), dtype=torch.bfloat16, device=dev)
    ws = torch.zeros(lib.sd_attention_workspace_bytes(1, H, dh, cap), dtype=torch.uint8, device=dev)
    tk, tv = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
    L.call("sd_make_slot_tmap", L.ptr(pk), Ln, Hk, cap, dh, tk)
    L.call("sd_make_slot_tmap", L.ptr(pv), Ln, Hk, cap, dh, tv)
    res = {}
    for name, maps in (("tensor_core", (tk, tv)), ("cuda_core", (None, None))):
        def run():
            for l in range(Ln):
                L.call("sd_attention", L.ptr(q), L.SD_BF16, 1, H, Hk, dh, 1, L.ptr(pk[l]), L.ptr(pv[l]), L.SD_BF16,
                       cap * dh, cap, L.ptr(rank[l]), L.ptr(cos_t), L.ptr(sin_t), L.ptr(kt), L.ptr(vt), dh, None,
                       0, None, None, maps[0], maps[1], l, Hk, L.ptr(out), L.SD_BF16, L.ptr(ws), ws.numel(),
                       L.stream())
        t = graph_time(run, a.reps) / Ln
        alg = 2 * (cap + 1) * Hk * dh * 2 + 2 * H * dh * 2
        res[name] = {"us": t * 1e6, "GB/s": alg / t / 1e9, "frac": alg / t / 1e9 / 6535.7}
    print(json.dumps({"H": H, "Hk": Hk, "slots": cap, **res}))


if __name__ == "__main__":
    main()
