"""Debug: per-row error of the tcgen05 verify kernel vs fp64 attention."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2502_18890_b200 import FullCache, _lib as L  # noqa: E402
from paper_2502_18890_b200.model import mask_bits_from_bool  # noqa: E402

ctx, T, Hk, force = [int(x) for x in sys.argv[1:5]]
H, dh, G = 4 * Hk, 128, 4
g = np.random.default_rng(0)
F = FullCache(1, Hk, dh, capacity=ctx + T + 64, dtype=torch.bfloat16)
F.k_rot.copy_(torch.as_tensor(g.normal(size=F.k_rot.shape), dtype=torch.bfloat16))
F.v.copy_(torch.as_tensor(g.normal(size=F.v.shape), dtype=torch.bfloat16))
q = torch.as_tensor(g.normal(size=(T, H, dh)) * 2 / np.sqrt(dh), dtype=torch.bfloat16, device="cuda")
mask = np.tril(np.ones((T, T), dtype=bool))
bits = torch.as_tensor(mask_bits_from_bool(mask), device="cuda")
out = torch.empty((T, H * dh), dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(L.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device="cuda")
L.call("sd_debug_tc_trace", None, force)
L.call("sd_attention", L.ptr(q), 1, T, H, Hk, dh, 0, L.ptr(F.k_rot[0]), L.ptr(F.v[0]), 1, F.head_stride, ctx, None,
       None, None, F.k_rot[0, :, ctx:].data_ptr(), F.v[0, :, ctx:].data_ptr(), F.head_stride, L.ptr(bits),
       L.MASK_WORDS, None, None, F.tmaps[0], F.tmaps[1], 0, 0, L.ptr(out), 1, L.ptr(ws), ws.numel(), L.stream())
got = out.double().cpu().numpy().reshape(T, H, dh)
K = F.k_rot[0].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
V = F.v[0].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
qq = q.double().cpu().numpy()
vis = np.zeros((T, ctx + T), dtype=bool)
vis[:, :ctx] = True
vis[:, ctx:] = mask
s = np.einsum("tkgd,nkd->tkgn", qq.reshape(T, Hk, G, dh), K)
s = np.where(vis[:, None, None, :], s, -np.inf)
w = np.exp(s - s.max(-1, keepdims=True))
w /= w.sum(-1, keepdims=True)
want = np.einsum("tkgn,nkd->tkgd", w, V).reshape(T, H, dh)
err = np.abs(got - want).max(-1)  # [T, H]
for kv in range(Hk):
    rows = [(t * G + gg, err[t, kv * G + gg]) for t in range(T) for gg in range(G)]
    bad = [r for r, e in rows if e > 0.02]
    print(f"kv head {kv}: bad rows {len(bad)} / {len(rows)}; first bad: {bad[:12]} max err {max(e for _, e in rows):.3f}")
