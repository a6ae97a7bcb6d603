"""Verify attention (tcgen05 + merge) timing at the BASELINE configs' head layouts
(tools/gpu_minchunk.sh): ctx, T, H, Hk per line; CUDA events over a graph of 20 calls (same K/V: L2-warm for small ctx)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2502_18890_b200 import FullCache, _lib as L
from paper_2502_18890_b200.model import mask_bits_from_bool
SHAPES = [(12048, 42, 12, 2), (2048, 42, 12, 2), (4096, 41, 32, 8), (12048, 41, 32, 8), (54096, 41, 32, 8),
          (54096, 42, 40, 8)]
import os
if os.environ.get('TC_SHAPES'):
    SHAPES = [tuple(int(x) for x in t.split(',')) for t in os.environ['TC_SHAPES'].split(';')]
for (ctx, T, H, Hk) in SHAPES:
    dh = 128
    F = FullCache(1, Hk, dh, capacity=ctx + T + 64, dtype=torch.bfloat16)
    F.k_rot.normal_(); F.v.normal_()
    q = (torch.randn((T, H, dh), device="cuda") * 0.1).to(torch.bfloat16)
    bits = torch.as_tensor(mask_bits_from_bool(np.tril(np.ones((T, T), dtype=bool))), device="cuda")
    out = torch.empty((T, H * dh), dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(L.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device="cuda")
    def run():
        L.call("sd_attention", L.ptr(q), 1, T, H, Hk, dh, 0, L.ptr(F.k_rot[0]), L.ptr(F.v[0]), 1, F.head_stride, ctx, None,
               None, None, F.k_rot[0, :, ctx:].data_ptr(), F.v[0, :, ctx:].data_ptr(), F.head_stride, L.ptr(bits),
               L.MASK_WORDS, None, None, F.tmaps[0], F.tmaps[1], 0, Hk, L.ptr(out), 1, L.ptr(ws), ws.numel(), L.stream())
    for _ in range(3): run()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):  # graph replay: device time, no per-call host overhead
        with torch.cuda.graph(g, stream=st):
            for _ in range(20): run()
        g.replay(); torch.cuda.synchronize()
        best = 1e9
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 20 * 1000)
    byt = 2 * ctx * Hk * dh * 2
    print(f"ctx={ctx} T={T} H={H} Hk={Hk}: {best:.1f} us  {byt / best / 1e3:.0f} GB/s")
