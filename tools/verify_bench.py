"""Verification attention alone (tcgen05 path): correctness vs torch fp32 on a
small case, then CUDA-graph timing at cfg shapes, incl. the engine's padded
launch (T_host = 101 with a device-resident live row count).

    python tools/verify_bench.py          (SD_VERIFY_V1=1: round-1 kernel)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_18890_b200 import FullCache, _lib as L  # noqa: E402
from paper_2502_18890_b200.model import mask_bits_from_bool  # noqa: E402


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


def setup(ctx, T_host, Hk, G, layers=1, seed=0):
    H, dh = G * Hk, 128
    F = FullCache(layers, Hk, dh, capacity=ctx + T_host + 64, dtype=torch.bfloat16)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    F.k_rot.normal_(generator=gen)
    F.v.normal_(generator=gen)
    q = (torch.randn((T_host, H, dh), device="cuda", generator=gen) * 0.15).to(torch.bfloat16)
    par = [-1] + [(i - 1) // 3 for i in range(1, T_host)]  # a ternary tree
    m = np.zeros((T_host, T_host), dtype=bool)
    for i in range(T_host):
        j = i
        while j >= 0:
            m[i, j] = True
            j = par[j]
    bits = torch.as_tensor(mask_bits_from_bool(m), device="cuda")
    out = torch.zeros((T_host, H * dh), dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(L.load().sd_attention_workspace_bytes(T_host, H, dh, ctx), dtype=torch.uint8, device="cuda")
    return dict(F=F, q=q, bits=bits, m=m, out=out, ws=ws, H=H, dh=dh)


def call(S, ctx, T_host, Hk, layer=0, rows_dev=None):
    F, dh, H = S["F"], S["dh"], S["H"]
    L.call("sd_attention", L.ptr(S["q"]), 1, T_host, H, Hk, dh, 0, L.ptr(F.k_rot[layer]), L.ptr(F.v[layer]), 1,
           F.head_stride, ctx, None, None, None, F.k_rot[layer, :, ctx:].data_ptr(), F.v[layer, :, ctx:].data_ptr(),
           F.head_stride, L.ptr(S["bits"]), L.MASK_WORDS, L.ptr(rows_dev), None, F.tmaps[0], F.tmaps[1], layer, 0,
           L.ptr(S["out"]), 1, L.ptr(S["ws"]), S["ws"].numel(), L.stream())


def reference(S, ctx, T, Hk, G):
    F, dh = S["F"], S["dh"]
    q = S["q"][:T].float()  # [T, H, dh]
    K = F.k_rot[0, :, :ctx + T].float()  # [Hk, ctx+T, dh]
    V = F.v[0, :, :ctx + T].float()
    outs = []
    for h in range(G * Hk):
        kv = h // G
        s = q[:, h] @ K[kv].T  # [T, ctx+T]
        vis = torch.ones_like(s, dtype=torch.bool)
        vis[:, ctx:] = torch.as_tensor(S["m"][:T, :T], device="cuda")
        s = s.masked_fill(~vis, float("-inf"))
        outs.append(torch.softmax(s, dim=-1) @ V[kv])
    return torch.stack(outs, dim=1).reshape(T, -1)


def main():
    res = {"kernel": "v1" if os.environ.get("SD_VERIFY_V1") == "1" else "cluster"}
    # correctness: live T < padded T through rows_dev, and T_host == T
    for (ctx, T, T_host, Hk, G) in [(5000, 41, 101, 8, 4), (3000, 41, 41, 8, 4), (2500, 101, 101, 2, 6),
                                    (700, 20, 20, 32, 1), (9000, 64, 101, 8, 5)]:
        S = setup(ctx, T_host, Hk, G)
        rows = torch.tensor([T], dtype=torch.int32, device="cuda")
        call(S, ctx, T_host, Hk, rows_dev=rows if T != T_host else None)
        torch.cuda.synchronize()
        want = reference(S, ctx, T, Hk, G)
        got = S["out"][:T].float()
        err = float((got - want).abs().max() / want.abs().max())
        res[f"err ctx{ctx} T{T}/{T_host} Hk{Hk} G{G}"] = err
    # timing at cfg shapes
    for (ctx, T, T_host, Hk, G, name) in [(54096, 41, 41, 8, 4, "cfg3 T41"), (54096, 41, 101, 8, 4, "cfg3 T41 pad101"),
                                          (54096, 101, 101, 8, 4, "cfg3 T101"), (104000, 41, 101, 8, 4, "cfg3 104K T41"),
                                          (12048, 41, 101, 2, 6, "cfg2 T41"), (54096, 41, 101, 32, 1, "cfg4 T41"),
                                          (54096, 41, 101, 8, 5, "cfg5 T41")]:
        Ln = 4
        S = setup(ctx, T_host, Hk, G, layers=Ln)
        rows = torch.tensor([T], dtype=torch.int32, device="cuda")
        rd = rows if T != T_host else None
        t = graph_time(lambda: [call(S, ctx, T_host, Hk, layer=l, rows_dev=rd) for l in range(Ln)], 10) / Ln
        H = G * Hk
        alg = 2 * ctx * Hk * 128 * 2 + 2 * T * H * 128 * 2 + 2 * T * Hk * 128 * 2
        res[name] = {"us": round(t * 1e6, 2), "GB/s": round(alg / t / 1e9), "frac": round(alg / t / 1e9 / 6535.7, 3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
