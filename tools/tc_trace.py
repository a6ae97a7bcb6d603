"""Debug: event timeline of the tcgen05 verification kernel's first CTA.

    python tools/tc_trace.py [ctx] [T]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_18890_b200 import FullCache, _lib as L  # noqa: E402
from paper_2502_18890_b200.model import mask_bits_from_bool  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 54096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 41
Hk = int(sys.argv[3]) if len(sys.argv) > 3 else 8
force = int(sys.argv[4]) if len(sys.argv) > 4 else 0
H, dh = 4 * Hk, 128
F = FullCache(1, Hk, dh, capacity=ctx + T + 64, dtype=torch.bfloat16)
F.k_rot.normal_()
F.v.normal_()
q = (torch.randn((T, H, dh), device="cuda") * 0.1).to(torch.bfloat16)
bits = torch.as_tensor(mask_bits_from_bool(np.tril(np.ones((T, T), dtype=bool))), device="cuda")
out = torch.empty((T, H * dh), dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(L.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device="cuda")
tr = torch.zeros(4 * 64 * 8 + 64 + 2 * 1024, dtype=torch.int64, device="cuda")


def run():
    L.call("sd_attention", L.ptr(q), 1, T, H, Hk, dh, 0, L.ptr(F.k_rot[0]), L.ptr(F.v[0]), 1, F.head_stride, ctx, None,
           None, None, F.k_rot[0, :, ctx:].data_ptr(), F.v[0, :, ctx:].data_ptr(), F.head_stride, L.ptr(bits),
           L.MASK_WORDS, None, None, F.tmaps[0], F.tmaps[1], 0, 0, L.ptr(out), 1, L.ptr(ws), ws.numel(), L.stream())


L.call("sd_debug_tc_trace", None, force)
for _ in range(3):
    run()
L.call("sd_debug_tc_trace", L.ptr(tr), force)
run()
torch.cuda.synchronize()
L.call("sd_debug_tc_trace", None, force)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(f"ctx={ctx} T={T}: {e0.elapsed_time(e1) / 10 * 1000:.1f} us per call")
allt = tr.cpu().numpy()
t = allt[:4 * 64 * 8].reshape(4, 64, 8)
cta = allt[4 * 64 * 8 + 64:].reshape(-1, 2)
cta = cta[cta[:, 1] > 0]
base = t[t > 0].min()
print("cta(0,0,0) milestones [entry, q staged, tmem+sync, softmax loop done, o_final, epilogue done, exit]:",
      [int(x - base) if x else None for x in t[0, 60, :7]])
names = {0: ["-", "K issued", "V issued"], 1: ["qk wait", "k_full ok", "qk issued", "v wait", "p ok", "-", "pv issued"],
         2: ["s wait", "s ok", "exp done", "rescaled", "p arrive"], 3: ["s wait", "s ok", "exp done", "rescaled", "p arrive"]}
for j in list(range(0, 6)) + list(range(20, 24)):
    row = []
    for role in range(4):
        for ev, nm in enumerate(names[role]):
            v = t[role, j, ev]
            if v:
                row.append(f"{['P', 'M', 'S0', 'S1'][role]}.{nm}={v - base}")
    print(f"tile {j:2d}: " + "  ".join(row))


print("\nper-tile deltas (cycles), tiles 20..27:")
print(" j | S0: wait  ld->exp  exp->resc  resc->P | S1: wait  ld->exp  exp->resc  resc->P | M: v->P  P->PV | S0 period")
prev = None
for j in range(20, 28):
    s0, s1, m = t[2, j], t[3, j], t[1, j]
    per = (s0[4] - prev) if prev is not None else 0
    prev = s0[4]
    print(f"{j:2d} | {s0[1]-s0[0]:6d} {s0[2]-s0[1]:7d} {s0[3]-s0[2]:9d} {s0[4]-s0[3]:8d} | "
          f"{s1[1]-s1[0]:6d} {s1[2]-s1[1]:7d} {s1[3]-s1[2]:9d} {s1[4]-s1[3]:8d} | {m[4]-m[3]:5d} {m[6]-m[4]:5d} | {per}")

print("\nK/V stream (slot q = tiles 2q, 2q+1): issue -> issuer-needs -> landed-seen; lead = need - issue, stall = seen - need")
for q in range(4, 24):
    j = 2 * q
    ki, vi = t[0, q, 1], t[0, q, 2]
    kw, kok = t[1, j, 0], t[1, j, 1]
    vw, vok = t[1, j, 3], t[1, j, 4]
    if ki and kw:
        print(f"slot {q:2d}: K issue {ki - base:7d} need {kw - base:7d} seen {kok - base:7d} lead {kw - ki:6d} stall {kok - kw:5d}"
              f" | V issue {vi - base:7d} need {vw - base:7d} (P ok {vok - base:7d}) lead {vw - vi:6d}")

if len(cta):
    t0 = cta[:, 0].min()
    st, en = (cta[:, 0] - t0) / 1e3, (cta[:, 1] - t0) / 1e3
    print(f"\nper-CTA (us from first start, {len(cta)} CTAs): start min {st.min():.1f} med {np.median(st):.1f} max {st.max():.1f}; "
          f"end min {en.min():.1f} med {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f}; "
          f"duration med {np.median(en - st):.1f} max {(en - st).max():.1f}")
    order = np.argsort(-en)[:8]
    print("latest CTAs (index, start, end):", [(int(i), round(float(st[i]), 1), round(float(en[i]), 1)) for i in order])
