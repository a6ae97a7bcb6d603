"""Sample SM clocks (nvidia-smi) while the verification attention runs back to
back for a few seconds: is the tensor-heavy kernel clock- or power-limited?"""
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import FullCache, _lib as L  # noqa: E402
from paper_2502_18890_b200.model import mask_bits_from_bool  # noqa: E402

ctx, T, Hk = 54096, 41, 8
H, dh = 4 * Hk, 128
F = FullCache(1, Hk, dh, capacity=ctx + T + 64, dtype=torch.bfloat16)
F.k_rot.normal_()
F.v.normal_()
q = (torch.randn((T, H, dh), device="cuda") * 0.1).to(torch.bfloat16)
bits = torch.as_tensor(mask_bits_from_bool(np.tril(np.ones((T, T), dtype=bool))), device="cuda")
out = torch.empty((T, H * dh), dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(L.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device="cuda")


def run():
    L.call("sd_attention", L.ptr(q), 1, T, H, Hk, dh, 0, L.ptr(F.k_rot[0]), L.ptr(F.v[0]), 1, F.head_stride, ctx, None,
           None, None, F.k_rot[0, :, ctx:].data_ptr(), F.v[0, :, ctx:].data_ptr(), F.head_stride, L.ptr(bits),
           L.MASK_WORDS, None, None, F.tmaps[0], F.tmaps[1], 0, 0, L.ptr(out), 1, L.ptr(ws), ws.numel(), L.stream())


g = torch.cuda.CUDAGraph()
run()
torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(200):
            run()
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader",
                        "-lms", "50"], stdout=subprocess.PIPE, text=True)
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    g.replay()
    n += 200
e1.record()
torch.cuda.synchronize()
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
print(f"{n} launches, {e0.elapsed_time(e1) / n * 1e3:.1f} us each (graph replay)")
for l in lines[::8]:
    print(l)
