"""Per-kernel parity of the CUDA path against the CPU oracle (oracle/) and the
reference's golden vectors. Integer outputs are compared bit-exactly; fp32
paths at 1e-5 relative, bf16 paths at 1e-2 relative (north star tolerance)."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import engine as OE
from oracle import kvcache as OK
from oracle import model as OM
from oracle import ngram as ON
from oracle import sampling as OS
from oracle import tree as OT

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
J = json.load(open(os.path.join(HERE, "golden.json")))
A = np.load(os.path.join(HERE, "golden.npz"))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_18890_b200 import _lib
    _lib.require_cuda()
    return _lib


def rope_np(x, pos, dh):
    inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
    return OM.rope(x, pos, inv)


def attend_oracle(q, K, V, vis):
    """q [T, H, dh] (rotated, scaled); K, V [n, Hk, dh]; vis [T, n] bool."""
    T, H, dh = q.shape
    Hk = K.shape[1]
    G = H // Hk
    s = np.einsum("tkgd,nkd->tkgn", q.reshape(T, Hk, G, dh), K)
    s = np.where(vis[:, None, None, :], s, -np.inf)
    s = np.exp(s - s.max(-1, keepdims=True))
    w = s / s.sum(-1, keepdims=True)
    return np.einsum("tkgn,nkd->tkgd", w, V).reshape(T, H, dh)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("ctx,T,H,Hk,dh", [(0, 5, 4, 2, 8), (37, 12, 8, 2, 32), (700, 41, 32, 8, 128),
                                            (3000, 101, 8, 8, 64), (5, 1, 4, 1, 16), (300, 3, 12, 2, 128)])
def test_verify_attention_tree(lib, dtype, ctx, T, H, Hk, dh):
    g = np.random.default_rng(ctx + T)
    dev = torch.device("cuda")
    cap = ctx + T + 3
    K = g.normal(size=(Hk, cap, dh))
    Vv = g.normal(size=(Hk, cap, dh))
    q = g.normal(size=(T, H, dh)) / np.sqrt(dh)
    # random tree over T rows (row 0 root)
    parent = [-1] + [int(g.integers(0, i)) for i in range(1, T)]
    mask = np.zeros((T, T), dtype=bool)
    for i in range(T):
        j = i
        while j >= 0:
            mask[i, j] = True
            j = parent[j]
    from paper_2502_18890_b200.model import mask_bits_from_bool
    bits = torch.as_tensor(mask_bits_from_bool(mask), device=dev)
    kt = torch.as_tensor(K, dtype=dtype, device=dev).contiguous()
    vt = torch.as_tensor(Vv, dtype=dtype, device=dev).contiguous()
    qt = torch.as_tensor(q, dtype=dtype, device=dev).contiguous()
    out = torch.empty((T, H * dh), dtype=dtype, device=dev)
    ws = torch.zeros(lib.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device=dev)
    kd = lib.dcode(dtype)
    lib.call("sd_attention", lib.ptr(qt), kd, T, H, Hk, dh, 0, lib.ptr(kt), lib.ptr(vt), kd, cap * dh, ctx, None,
             None, None, kt[:, ctx:].data_ptr(), vt[:, ctx:].data_ptr(), cap * dh, lib.ptr(bits), lib.MASK_WORDS,
             None, None, None, None, 0, 0, lib.ptr(out), kd, lib.ptr(ws), ws.numel(), lib.stream())
    # oracle on the same (rounded) inputs
    Kr = kt.double().cpu().numpy().transpose(1, 0, 2)
    Vr = vt.double().cpu().numpy().transpose(1, 0, 2)
    qr = qt.double().cpu().numpy()
    vis = np.zeros((T, ctx + T), dtype=bool)
    vis[:, :ctx] = True
    vis[:, ctx:] = mask
    want = attend_oracle(qr, Kr[: ctx + T], Vr[: ctx + T], vis)
    got = out.double().cpu().numpy().reshape(T, H, dh)
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol)


@pytest.mark.parametrize("ctx,T,H,Hk,layer", [(64, 1, 32, 8, 0), (100, 5, 32, 8, 1), (700, 41, 32, 8, 2),
                                               (4096, 41, 32, 8, 0), (3000, 101, 32, 8, 1), (1500, 20, 40, 8, 2),
                                               (20000, 41, 32, 8, 1), (900, 70, 32, 32, 0)])
def test_verify_attention_tcgen05(lib, ctx, T, H, Hk, layer):
    """tcgen05/TMA/TMEM path (bf16, dh=128) vs the fp64 oracle and vs the CUDA-core path."""
    from paper_2502_18890_b200 import FullCache
    from paper_2502_18890_b200.model import mask_bits_from_bool
    dev = torch.device("cuda")
    g = np.random.default_rng(ctx * 7 + T)
    dh, Lr = 128, 3
    cap = ctx + T + 70
    F = FullCache(Lr, Hk, dh, capacity=cap, dtype=torch.bfloat16)
    assert F.tmaps is not None
    F.k_rot.copy_(torch.as_tensor(g.normal(size=(Lr, Hk, cap, dh)), dtype=torch.bfloat16))
    F.v.copy_(torch.as_tensor(g.normal(size=(Lr, Hk, cap, dh)), dtype=torch.bfloat16))
    parent = [-1] + [int(g.integers(0, i)) for i in range(1, T)]
    mask = np.zeros((T, T), dtype=bool)
    for i in range(T):
        j = i
        while j >= 0:
            mask[i, j] = True
            j = parent[j]
    bits = torch.as_tensor(mask_bits_from_bool(mask), device=dev)
    qt = torch.as_tensor(g.normal(size=(T, H, dh)) * 2.0 / np.sqrt(dh), dtype=torch.bfloat16, device=dev)
    outs = []
    for tm in (F.tmaps, (None, None)):
        out = torch.empty((T, H * dh), dtype=torch.bfloat16, device=dev)
        ws = torch.zeros(lib.load().sd_attention_workspace_bytes(T, H, dh, ctx), dtype=torch.uint8, device=dev)
        lib.call("sd_attention", lib.ptr(qt), 1, T, H, Hk, dh, 0, lib.ptr(F.k_rot[layer]), lib.ptr(F.v[layer]), 1,
                 F.head_stride, ctx, None, None, None, F.k_rot[layer, :, ctx:].data_ptr(),
                 F.v[layer, :, ctx:].data_ptr(), F.head_stride, lib.ptr(bits), lib.MASK_WORDS, None, None, tm[0], tm[1],
                 layer, 0, lib.ptr(out), 1, lib.ptr(ws), ws.numel(), lib.stream())
        outs.append(out.double().cpu().numpy().reshape(T, H, dh))
    Kr = F.k_rot[layer].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
    Vr = F.v[layer].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
    vis = np.zeros((T, ctx + T), dtype=bool)
    vis[:, :ctx] = True
    vis[:, ctx:] = mask
    want = attend_oracle(qt.double().cpu().numpy(), Kr, Vr, vis)
    np.testing.assert_allclose(outs[0], want, rtol=1e-2, atol=1e-2)
    np.testing.assert_allclose(outs[0], outs[1], rtol=1e-2, atol=1e-2)
    assert np.max(np.abs(outs[0] - want)) < 1.5e-2


@pytest.mark.parametrize("tc", [True, False])
@pytest.mark.parametrize("ctx", [70, 3000, 20000])
def test_attention_ctx_dev_matches_host_ctx(lib, tc, ctx):
    """Device-resident context (graph replay): ctx read on device with a larger
    host upper bound, tree rows right after the live rows, stale workspace —
    same result as the host-ctx call (bitwise on the CUDA-core path)."""
    from paper_2502_18890_b200 import FullCache
    from paper_2502_18890_b200.model import mask_bits_from_bool
    dev = torch.device("cuda")
    g = np.random.default_rng(ctx)
    T, H, Hk, dh, Lr, layer = 41, 32, 8, 128, 2, 1
    cap = 24000
    F = FullCache(Lr, Hk, dh, capacity=cap, dtype=torch.bfloat16)
    F.k_rot.normal_()
    F.v.normal_()
    parent = [-1] + [int(g.integers(0, i)) for i in range(1, T)]
    mask = np.zeros((T, T), dtype=bool)
    for i in range(T):
        j = i
        while j >= 0:
            mask[i, j] = True
            j = parent[j]
    bits = torch.as_tensor(mask_bits_from_bool(mask), device=dev)
    qt = (torch.randn((T, H, dh), device=dev) * 0.2).to(torch.bfloat16)
    tm = F.tmaps if tc else (None, None)
    ctx_dev = torch.tensor([ctx], dtype=torch.int32, device=dev)
    upper = cap - T
    ws = torch.full((lib.load().sd_attention_workspace_bytes(T, H, dh, upper),), 255, dtype=torch.uint8, device=dev)
    ws[:4096] = 0  # SD_ATTN_WS_HEAD: the counter head is zero between calls; the rest is stale
    outs = []
    for mode in ("host", "dev"):
        out = torch.empty((T, H * dh), dtype=torch.bfloat16, device=dev)
        if mode == "host":
            lib.call("sd_attention", lib.ptr(qt), 1, T, H, Hk, dh, 0, lib.ptr(F.k_rot[layer]), lib.ptr(F.v[layer]), 1,
                     F.head_stride, ctx, None, None, None, F.k_rot[layer, :, ctx:].data_ptr(),
                     F.v[layer, :, ctx:].data_ptr(), F.head_stride, lib.ptr(bits), lib.MASK_WORDS, None, None, tm[0],
                     tm[1], layer, 0, lib.ptr(out), 1, lib.ptr(ws), ws.numel(), lib.stream())
        else:
            lib.call("sd_attention", lib.ptr(qt), 1, T, H, Hk, dh, 0, lib.ptr(F.k_rot[layer]), lib.ptr(F.v[layer]), 1,
                     F.head_stride, upper, None, None, None, None, None, F.head_stride, lib.ptr(bits), lib.MASK_WORDS,
                     None, lib.ptr(ctx_dev), tm[0], tm[1], layer, 0, lib.ptr(out), 1, lib.ptr(ws), ws.numel(),
                     lib.stream())
        outs.append(out.float())
    assert torch.isfinite(outs[1]).all()
    if tc:
        torch.testing.assert_close(outs[1], outs[0], rtol=1e-2, atol=1e-2)
    Kr = F.k_rot[layer].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
    Vr = F.v[layer].double().cpu().numpy().transpose(1, 0, 2)[: ctx + T]
    vis = np.zeros((T, ctx + T), dtype=bool)
    vis[:, :ctx] = True
    vis[:, ctx:] = mask
    want = attend_oracle(qt.double().cpu().numpy(), Kr, Vr, vis)
    np.testing.assert_allclose(outs[1].double().cpu().numpy().reshape(T, H, dh), want, rtol=1e-2, atol=1e-2)


def test_attention_rows_dev_padding(lib):
    dev = torch.device("cuda")
    T, Tl, H, Hk, dh, ctx = 16, 7, 8, 2, 64, 200
    g = np.random.default_rng(3)
    cap = ctx + T
    kt = torch.as_tensor(g.normal(size=(Hk, cap, dh)), dtype=torch.float32, device=dev)
    vt = torch.as_tensor(g.normal(size=(Hk, cap, dh)), dtype=torch.float32, device=dev)
    qt = torch.as_tensor(g.normal(size=(T, H, dh)) * 0.1, dtype=torch.float32, device=dev)
    rows = torch.tensor([Tl], dtype=torch.int32, device=dev)
    outs = []
    for rd in (rows, None):
        TT = T if rd is not None else Tl
        out = torch.full((TT, H * dh), 7.0, dtype=torch.float32, device=dev)
        ws = torch.zeros(lib.load().sd_attention_workspace_bytes(TT, H, dh, ctx), dtype=torch.uint8, device=dev)
        lib.call("sd_attention", lib.ptr(qt), 0, TT, H, Hk, dh, 0, lib.ptr(kt), lib.ptr(vt), 0, cap * dh, ctx, None,
                 None, None, kt[:, ctx:].data_ptr(), vt[:, ctx:].data_ptr(), cap * dh, None, 0, lib.ptr(rd),
                 None, None, None, 0, 0, lib.ptr(out), 0, lib.ptr(ws), ws.numel(), lib.stream())
        outs.append(out)
    assert torch.equal(outs[0][:Tl], outs[1])
    assert torch.all(outs[0][Tl:] == 0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("H,Hk,dh,cap,hi", [(8, 2, 32, 300, 260), (32, 8, 128, 4200, 4100), (40, 8, 128, 700, 650),
                                            (16, 16, 64, 300, 290), (12, 2, 128, 2100, 2050), (16, 8, 128, 300, 290),
                                            (24, 8, 128, 130, 5)])
def test_draft_attention_rank_rope_with_holes(lib, dtype, H, Hk, dh, cap, hi):
    dev = torch.device("cuda")
    g = np.random.default_rng(11)
    ranks = -np.ones(hi, dtype=np.int32)
    live = np.sort(g.choice(hi, size=int(hi * 0.8), replace=False))
    perm = g.permutation(len(live))
    ranks[live] = perm  # arbitrary rank per live slot
    Kraw = g.normal(size=(Hk, cap, dh))
    V = g.normal(size=(Hk, cap, dh))
    m = len(live)
    from paper_2502_18890_b200 import ModelConfig, TinyTransformer
    mdl = TinyTransformer(ModelConfig(vocab_size=16, hidden_dim=H * dh, num_heads=H, num_kv_heads=Hk,
                                      max_positions=4096), dtype=dtype)
    q_raw = g.normal(size=(1, H, dh))
    k_self = g.normal(size=(1, Hk, dh))
    v_self = g.normal(size=(1, Hk, dh))
    q = rope_np(q_raw, [m], dh) / np.sqrt(dh)
    ks = rope_np(k_self, [m], dh)
    pk = torch.as_tensor(Kraw, dtype=dtype, device=dev)
    pv = torch.as_tensor(V, dtype=dtype, device=dev)
    rk = torch.as_tensor(ranks, device=dev)
    qt = torch.as_tensor(q, dtype=dtype, device=dev)
    kt = torch.as_tensor(ks.transpose(1, 0, 2), dtype=dtype, device=dev).contiguous()
    vt = torch.as_tensor(v_self.transpose(1, 0, 2), dtype=dtype, device=dev).contiguous()
    outs = []
    out = torch.empty((1, H * dh), dtype=dtype, device=dev)
    mdl.attention(qt, 1, 1, pk, pv, cap * dh, hi, rk, kt, vt, dh, None, None, out)
    outs.append(out)
    if dtype == torch.bfloat16 and dh == 128:
        # the product path: TMA slot descriptors -> tensor-core draft kernel
        import ctypes
        tk, tv = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
        lib.call("sd_make_slot_tmap", lib.ptr(pk), 1, Hk, cap, dh, tk)
        lib.call("sd_make_slot_tmap", lib.ptr(pv), 1, Hk, cap, dh, tv)
        out2 = torch.empty((1, H * dh), dtype=dtype, device=dev)
        mdl.attention(qt, 1, 1, pk, pv, cap * dh, hi, rk, kt, vt, dh, None, None, out2, (tk, tv), 0)
        outs.append(out2)
    # oracle: keys sorted by rank, rotated at rank
    order = live[np.argsort(ranks[live])]
    Kr = pk.double().cpu().numpy()[:, order].transpose(1, 0, 2)
    Vr = pv.double().cpu().numpy()[:, order].transpose(1, 0, 2)
    Krot = rope_np(Kr, np.arange(m), dh)
    Kall = np.concatenate([Krot, kt.double().cpu().numpy().transpose(1, 0, 2)])
    Vall = np.concatenate([Vr, vt.double().cpu().numpy().transpose(1, 0, 2)])
    want = attend_oracle(qt.double().cpu().numpy(), Kall, Vall, np.ones((1, m + 1), dtype=bool))
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    for o in outs:
        got = o.double().cpu().numpy().reshape(1, H, dh)
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("ctx", [1, 63, 5000, 54000])
def test_decode_attention_full_cache(lib, dtype, ctx):
    """T == 1 over the full cache (AR decode path) vs the oracle."""
    dev = torch.device("cuda")
    g = np.random.default_rng(ctx)
    H, Hk, dh = 32, 8, 128
    cap = ctx + 4
    kt = torch.as_tensor(g.normal(size=(Hk, cap, dh)), dtype=dtype, device=dev)
    vt = torch.as_tensor(g.normal(size=(Hk, cap, dh)), dtype=dtype, device=dev)
    qt = torch.as_tensor(g.normal(size=(1, H, dh)) * 2 / np.sqrt(dh), dtype=dtype, device=dev)
    out = torch.empty((1, H * dh), dtype=dtype, device=dev)
    ws = torch.zeros(lib.load().sd_attention_workspace_bytes(1, H, dh, ctx), dtype=torch.uint8, device=dev)
    kd = lib.dcode(dtype)
    lib.call("sd_attention", lib.ptr(qt), kd, 1, H, Hk, dh, 0, lib.ptr(kt), lib.ptr(vt), kd, cap * dh, ctx, None,
             None, None, kt[:, ctx:].data_ptr(), vt[:, ctx:].data_ptr(), cap * dh, None, 0, None, None, None, None, 0,
             0, lib.ptr(out), kd, lib.ptr(ws), ws.numel(), lib.stream())
    Kr = kt.double().cpu().numpy().transpose(1, 0, 2)[: ctx + 1]
    Vr = vt.double().cpu().numpy().transpose(1, 0, 2)[: ctx + 1]
    want = attend_oracle(qt.double().cpu().numpy(), Kr, Vr, np.ones((1, ctx + 1), dtype=bool))
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    np.testing.assert_allclose(out.double().cpu().numpy().reshape(1, H, dh), want, rtol=tol, atol=tol)


def test_importance_scores_golden(lib):
    from paper_2502_18890_b200 import importance_scores
    for gs in J["imp_groups"]:
        q, k = A[f"imp_q{gs}"], A[f"imp_k{gs}"]
        # dh = 5 is not a supported head size: pad to 8 with zeros (score unchanged)
        qp = np.zeros((q.shape[0], 8))
        qp[:, :5] = q
        kp = np.zeros(k.shape[:2] + (8,))
        kp[..., :5] = k
        got = importance_scores(qp, kp, gs).cpu().numpy()
        np.testing.assert_allclose(got, A[f"imp_s{gs}"], rtol=1e-5, atol=1e-5)


def _scored_partial(lib, scores, sink, budget):
    """PartialCache.build_topk over a 1-head fp32 full cache whose V rows hold
    their own position (so gathered data can be checked slot by slot)."""
    from paper_2502_18890_b200 import FullCache
    from paper_2502_18890_b200.kvcache import PartialCache
    Lr, nc = scores.shape
    n = nc + sink
    full = FullCache(Lr, 1, 8, capacity=n + 8, dtype=torch.float32)
    full.v[:, :, :n] = torch.arange(n, dtype=torch.float32, device="cuda").view(1, 1, n, 1)
    full.k_raw[:, :, :n] = -torch.arange(n, dtype=torch.float32, device="cuda").view(1, 1, n, 1)
    full.positions = list(range(n))
    part = PartialCache(sink, budget, Lr, 1, 8, torch.float32)
    part.build_topk(full, torch.as_tensor(scores, dtype=torch.float32, device="cuda"), n)
    return part


def _check_slots(part):
    """Slot invariants: ranks are the position order of live slots, data
    follows slots, holes are marked."""
    pos, rk = part.ppos.cpu().numpy(), part.ranks()
    for l in range(part.num_layers):
        live = [s for s in range(part.hi) if pos[l, s] >= 0]
        assert len(live) == part.count
        want = np.argsort(np.argsort([pos[l, s] for s in live]))
        assert [int(rk[l, s]) for s in live] == want.tolist()
        vals = part.pv[l, 0, live, 0].cpu().numpy()
        assert np.array_equal(vals, pos[l, live].astype(np.float32))


@pytest.mark.parametrize("trial", range(10))
def test_select_topk_golden(lib, trial):
    """Exact reference order (-score, pos) including ties (kvcache.py:286):
    fused select + gather (sd_partial_refresh on given scores)."""
    c = J["select"][trial]
    sc = A[f"sel{trial}_scores"].astype(np.float32)
    part = _scored_partial(lib, sc[:, : c["n"] - c["sink"]], c["sink"], c["budget"])
    assert part.positions == c["positions"]
    _check_slots(part)


def test_select_topk_large_random(lib):
    g = np.random.default_rng(5)
    Lr, n, sink, take = 3, 20000, 16, 4000
    sc = np.round(g.normal(size=(Lr, n)), 2).astype(np.float32)  # many ties
    part = _scored_partial(lib, sc, sink, sink + take)
    for l in range(Lr):
        want = list(range(sink)) + OK.select_body(sc[l].astype(np.float64), sink, sink + n, take)
        assert part.positions[l] == want
    _check_slots(part)


def _partial_case(L_, n, sink, budget):
    from paper_2502_18890_b200 import FullCache
    g = np.random.default_rng(n)
    full = FullCache(L_, 1, 8, capacity=n + 16, dtype=torch.float32)
    kr = g.normal(size=(L_, 1, n, 8))
    full.k_raw[:, :, :n] = torch.as_tensor(kr, dtype=torch.float32)
    full.v[:, :, :n] = torch.arange(n, dtype=torch.float32).view(1, 1, n, 1).expand(L_, 1, n, 8)
    full.positions = list(range(n))
    ofull = OK.FullCache(L_, 1, 8, cap=n + 16)
    ofull.k_raw[:, :n] = kr.transpose(0, 2, 1, 3)
    ofull.v[:, :n] = np.arange(n, dtype=np.float64)[None, :, None, None]
    ofull.positions = list(range(n))
    return full, ofull


def test_partial_admit_evict_matches_reference_semantics(lib):
    """test_kvcache.py:152-160 plus a long random admit/evict/refresh sequence."""
    from paper_2502_18890_b200 import kvcache as K
    full, ofull = _partial_case(1, 8, 2, 5)
    part = K.mirror_partial(full, 2, 5, upto=5)
    op = OK.mirror_partial(ofull, 2, 5, upto=5)
    assert part.positions == op.positions == [[0, 1, 4, 3, 2]]
    part.admit([5, 6], full)
    part.evict(protected=2)
    assert part.positions == [[0, 1, 5, 6, 4]]
    # long run against the oracle, two layers
    Lr, n = 2, 400
    full, ofull = _partial_case(Lr, n, 4, 24)
    part = K.mirror_partial(full, 4, 24, upto=10)
    op = OK.mirror_partial(ofull, 4, 24, upto=10)
    g = np.random.default_rng(9)
    cur = 10
    while cur < n - 8:
        if g.random() < 0.1 and cur >= 24:
            sc = np.round(g.normal(size=(Lr, cur - 4)), 1)
            part.build_topk(full, torch.as_tensor(sc, dtype=torch.float32, device="cuda"), cur)
            op = OK.prefill_partial(ofull, 4, 24, sc, upto=cur)
        a = int(g.integers(1, 5))
        part.admit_evict(cur, a, full, protected=a)
        op.admit(list(range(cur, cur + a)), ofull)
        OK.evict_to_budget(op, protected=a)
        cur += a
        assert part.positions == op.positions
        _check_slots(part)  # ranks are the position order of live slots; data follows slots


def test_reconcile_and_qsum(lib):
    from paper_2502_18890_b200 import FullCache
    from paper_2502_18890_b200 import _lib as Lb
    full = FullCache(2, 2, 8, capacity=64, dtype=torch.float32)
    for arr in (full.k_raw, full.k_rot, full.v):
        arr.copy_(torch.arange(arr.numel(), dtype=torch.float32, device="cuda").view(arr.shape))
    before = [t.clone() for t in (full.k_raw, full.k_rot, full.v)]
    base, keep = 10, [0, 2, 3, 7]
    res = torch.full((32,), -1, dtype=torch.int32)
    res[Lb.RES_ACCEPTED] = 4
    res[Lb.RES_KEEP:Lb.RES_KEEP + 4] = torch.tensor(keep)
    q_pre = torch.randn((2, 12, 4, 8), device="cuda")
    q_sum = torch.zeros((2, 4, 8), device="cuda")
    full.reconcile_device(base, res.cuda(), q_pre, 12, 4, q_sum)
    for b, t in zip(before, (full.k_raw, full.k_rot, full.v)):
        for i, k in enumerate(keep):
            assert torch.equal(t[:, :, base + i], b[:, :, base + k])
    want = sum(q_pre[:, k] for k in keep)
    torch.testing.assert_close(q_sum, want, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("trial", range(24))
def test_sampler_golden(lib, trial):
    from paper_2502_18890_b200 import sampling as S
    case = J["sampling"][trial]
    logits, members = A[f"samp{trial}_logits"], A[f"samp{trial}_members"]
    cfg = S.SamplerConfig(temperature=case["t"], theta=case["theta"], window=64, ctrl_style=case["ctrl"])
    probs = S.penalized_probs_masked(logits, members, cfg).cpu().numpy()
    np.testing.assert_allclose(probs, A[f"samp{trial}_probs"], rtol=1e-12, atol=1e-300)
    rules = [S.Truncation.min_p(0.1), S.Truncation.top_p(0.9), S.Truncation.eta(0.02),
             S.Truncation.top_p(0.5), S.Truncation.min_p(0.5)]
    for ri, rule in enumerate(rules):
        d = S.truncate(A[f"samp{trial}_probs"], rule).cpu().numpy()
        np.testing.assert_allclose(d, A[f"samp{trial}_trunc{ri}"], rtol=1e-12, atol=1e-300)
        got = [S.sample_at(A[f"samp{trial}_trunc{ri}"], pos, seed) for pos, seed in [(0, 0), (5, 1), (777, 3), (4096, 0)]]
        assert got == case["draws"][str(ri)]


def test_sampler_known_answers(lib):
    """test_sampling.py:128-213 restated against the device sampler."""
    from paper_2502_18890_b200 import sampling as S
    from paper_2502_18890_b200.rng import uniform_at
    assert np.allclose(S.truncate(np.array([0.5, 0.3, 0.2]), S.Truncation.top_p(1.0)).cpu().numpy(), [0.5, 0.3, 0.2])
    out = S.truncate(np.array([0.5, 0.04, 0.46]), S.Truncation.min_p(0.1)).cpu().numpy()
    assert out[1] == 0.0
    out = S.truncate(np.full(4, 0.25), S.Truncation.top_p(0.5)).cpu().numpy()
    assert np.count_nonzero(out) == 2 and np.allclose(out[out > 0], 0.5)
    out = S.truncate(np.full(4096, 1 / 4096), S.Truncation.eta(2e-4)).cpu().numpy()
    assert np.count_nonzero(out) >= 1 and abs(out.sum() - 1) < 1e-9
    d = np.array([0.3, 0.7])
    for seed in range(200):
        assert S.sample_at(d, 0, seed) == (0 if uniform_at(seed, 0) < 0.3 else 1)
    pm = np.zeros(16)
    pm[7] = 1.0
    assert all(S.sample_at(pm, p, s) == 7 for p in range(3) for s in range(3))


def test_verify_sampler_tree_rows_match_oracle_node_masks(lib):
    """Fused per-row window splice (engine.py:155-181) == oracle node_masks."""
    from paper_2502_18890_b200 import _lib as Lb
    from paper_2502_18890_b200.sampling import PenaltyWindow
    g = np.random.default_rng(21)
    V, W, depth = 64, 12, 4
    for trial in range(6):
        hist = g.integers(0, V, size=int(g.integers(0, 30))).tolist()
        ow = OS.PenaltyWindow(W, V)
        st = torch.zeros(16, dtype=torch.int64, device="cuda")
        dw = PenaltyWindow(W, V, state=st)
        for t in hist:
            ow.push(t)
        dw.push_many(hist)
        per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
        grams = [tuple([per_head[0][0]] + g.integers(0, V, size=3).tolist()) for _ in range(3)]
        tree = OT.build_tree(per_head, grams)
        masks = OS.node_masks(ow, tree.tokens, tree.parent, depth)
        T = 1 + len(tree)
        logits = g.normal(scale=2.0, size=(T, V))
        smp = OS.SamplerConfig(temperature=0.9, theta=1.3, window=W, truncation=OS.Truncation.top_p(0.8), seed=trial)
        n = 50 + trial
        want = []
        dists = OS.penalized_probs_masked(logits, masks, smp)
        for r in range(T):
            pos = n if r == 0 else n + tree.depth[r - 1] + 1
            want.append(OS.sample_at(OS.truncate(dists[r], smp.truncation), pos, smp.seed))
        # device: tree record + fused sampler
        rec = torch.zeros(Lb.tree_layout()["TOTAL"], dtype=torch.int32, device="cuda")
        flat = torch.tensor([t for c in per_head for t in c], dtype=torch.int32, device="cuda")
        gm = torch.tensor(grams, dtype=torch.int32, device="cuda").reshape(-1)
        Lb.call("sd_tree_build", Lb.ptr(flat), Lb.host_i32([1, 3, 3, 3]), 4, Lb.ptr(gm), None, len(grams), None, n - 1,
                Lb.ptr(rec), Lb.stream())
        lt = torch.as_tensor(logits, dtype=torch.float64, device="cuda")
        y = torch.full((T,), -1, dtype=torch.int32, device="cuda")
        probs = torch.empty((T, V), dtype=torch.float64, device="cuda")
        a = Lb.SampleArgs()
        a.rows, a.V, a.in_kind = T, V, Lb.IN_LOGITS_F64
        a.temperature, a.theta, a.ctrl_style = 0.9, 1.3, 0
        a.member_kind = Lb.MEMBER_TREE
        a.win_count, a.win_ring, a.state, a.window = Lb.ptr(dw.count), Lb.ptr(dw.ring), Lb.ptr(st), W
        a.tree, a.depth = Lb.ptr(rec), depth
        a.trunc_kind, a.trunc_value, a.eta_alpha = Lb.TRUNC_TOP_P, 0.8, -1.0
        a.seed, a.n = trial, n
        a.probs_out, a.token_out = Lb.ptr(probs), Lb.ptr(y)
        Lb.call("sd_sample_rows", Lb.ptr(lt), a, Lb.stream())
        np.testing.assert_allclose(probs.cpu().numpy(), dists, rtol=1e-12, atol=1e-300)
        assert y.cpu().tolist() == want


@pytest.mark.parametrize("trunc", ["min_p1", "min_p", "top_p"])
def test_cluster_sampler_matches_oracle(lib, trunc):
    """Engine-path sampler (8-CTA cluster per row, fp32 logits, token draw only)
    against the fp64 oracle: window splice per tree row (engine.py:155-181),
    Eq. 3 penalty, truncation, inverse CDF at uniform_at(seed, pos)
    (sampling.py:142-224), on logits exactly representable in fp32."""
    from paper_2502_18890_b200 import _lib as Lb
    from paper_2502_18890_b200.sampling import PenaltyWindow
    g = np.random.default_rng({"min_p1": 5, "min_p": 6, "top_p": 7}[trunc])
    V, W, depth = 5000, 48, 4
    code, val = {"min_p1": (Lb.TRUNC_MIN_P, 1.0), "min_p": (Lb.TRUNC_MIN_P, 0.1), "top_p": (Lb.TRUNC_TOP_P, 0.9)}[trunc]
    otr = {"min_p1": OS.Truncation.min_p(1.0), "min_p": OS.Truncation.min_p(0.1), "top_p": OS.Truncation.top_p(0.9)}[trunc]
    for trial in range(4):
        hist = g.integers(0, V, size=int(g.integers(10, 80))).tolist()
        ow = OS.PenaltyWindow(W, V)
        st = torch.zeros(16, dtype=torch.int64, device="cuda")
        dw = PenaltyWindow(W, V, state=st)
        for t in hist:
            ow.push(t)
        dw.push_many(hist)
        per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
        tree = OT.build_tree(per_head, [])
        masks = OS.node_masks(ow, tree.tokens, tree.parent, depth)
        T = 1 + len(tree)
        logits = g.normal(scale=3.0, size=(T, V)).astype(np.float32).astype(np.float64)
        smp = OS.SamplerConfig(temperature=0.9, theta=1.2, window=W, truncation=otr, seed=trial)
        n = 300 + trial
        dists = OS.penalized_probs_masked(logits, masks, smp)
        want = [OS.sample_at(OS.truncate(dists[r], smp.truncation), n if r == 0 else n + tree.depth[r - 1] + 1,
                             smp.seed) for r in range(T)]
        rec = torch.zeros(Lb.tree_layout()["TOTAL"], dtype=torch.int32, device="cuda")
        flat = torch.tensor([t for c in per_head for t in c], dtype=torch.int32, device="cuda")
        Lb.call("sd_tree_build", Lb.ptr(flat), Lb.host_i32([1, 3, 3, 3]), 4, None, None, 0, None, n - 1,
                Lb.ptr(rec), Lb.stream())
        lt = torch.as_tensor(logits, dtype=torch.float32, device="cuda")
        y = torch.full((T,), -1, dtype=torch.int32, device="cuda")
        a = Lb.SampleArgs()
        a.rows, a.V, a.in_kind = T, V, Lb.IN_LOGITS_F32
        a.temperature, a.theta, a.ctrl_style = 0.9, 1.2, 0
        a.member_kind = Lb.MEMBER_TREE
        a.win_count, a.win_ring, a.state, a.window = Lb.ptr(dw.count), Lb.ptr(dw.ring), Lb.ptr(st), W
        a.tree, a.depth = Lb.ptr(rec), depth
        a.trunc_kind, a.trunc_value, a.eta_alpha = code, val, -1.0
        a.seed, a.n = trial, n
        a.token_out = Lb.ptr(y)
        Lb.call("sd_sample_rows", Lb.ptr(lt), a, Lb.stream())  # cluster path: fp32, token only
        assert y.cpu().tolist() == want, (trunc, trial)


@pytest.mark.parametrize("V,widths", [(5000, [1, 3, 3, 3]), (20, [8, 5, 16, 2]), (151936, [16, 9, 4, 1]),
                                      (64, [16, 16, 16, 16])])
def test_draft_topw_matches_stable_argsort(lib, V, widths):
    """Per-head top-w over an 8-CTA cluster (vocabulary slices, some shorter than
    w): penalised scaled logits, ties -> lower id across slices (engine.py:207-215)."""
    g = np.random.default_rng(2)
    logits = g.normal(scale=3, size=(4, V)).astype(np.float32)
    logits[1, 17 % V] = logits[1, (4000 % V) or 1] = logits[1].max() + 1  # exact tie -> lower id first
    logits[2, V // 2: 2 * (V // 2)] = logits[2, : V // 2]  # equal logits in different slices (ties when both
    # have the same window membership)
    cnt = np.zeros(V, dtype=np.int32)
    cnt[g.integers(0, V, size=max(1, V // 16))] = 1
    smp = OS.SamplerConfig(temperature=1.0, theta=1.2, window=64)
    probs = OS.penalized_probs_masked(logits.astype(np.float64), np.broadcast_to(cnt > 0, (4, V)), smp)
    want = [int(t) for k in range(4) for t in np.argsort(-probs[k], kind="stable")[: widths[k]]]
    from paper_2502_18890_b200 import _lib as Lb
    out = torch.empty(sum(widths), dtype=torch.int32, device="cuda")
    lt = torch.as_tensor(logits, device="cuda")
    ct = torch.as_tensor(cnt, device="cuda")
    Lb.call("sd_draft_topw", Lb.ptr(lt), 4, V, Lb.ptr(ct), 1.0, 1.2, 0, Lb.host_i32(widths), Lb.ptr(out), Lb.stream())
    assert out.cpu().tolist() == want


@pytest.mark.parametrize("trial", range(6))
def test_ngram_golden(lib, trial):
    from paper_2502_18890_b200 import NGramTable
    c = J["ngram"][trial]
    tab = NGramTable(n=c["n"], k_max=64, capacity=8192, vocab_size=64)
    seq = []
    for chunk in c["ops"]:
        tab.update(chunk, seq[-(c["n"] - 1):] if c["n"] > 1 else [])
        seq.extend(chunk)
    assert len(tab) == c["size"]
    for f, want in c["retrieve"].items():
        assert [list(g) for g in tab.retrieve(int(f), 20)] == want
    for g, fr in c["freqs"]:
        assert tab.frequency(tuple(g)) == fr


def test_ngram_known_answers(lib):
    """test_ngram.py:19-98 restated."""
    from paper_2502_18890_b200 import NGramTable
    t = NGramTable(n=4, vocab_size=64)
    t.update([9], history_tail=[1, 2, 3])
    assert len(t) == 1 and t.frequency((1, 2, 3, 9)) == 1
    t = NGramTable(n=2, vocab_size=64)
    t.update([0, 1, 0, 1, 0, 1], history_tail=[])
    assert t.frequency((0, 1)) == 3 and t.frequency((1, 0)) == 2
    t = NGramTable(n=2, vocab_size=64)
    t.update([1, 2], [])
    t.update([1, 3], [])
    assert t.retrieve(1, 2) == [(1, 3), (1, 2)]
    t.update([1, 2], [])
    assert t.retrieve(1, 2) == [(1, 2), (1, 3)]
    with pytest.raises(ValueError):
        NGramTable(n=4, k_max=8, vocab_size=64).retrieve(0, 9)
    assert NGramTable(n=4, vocab_size=64).retrieve(0, 5) == []


@pytest.mark.parametrize("trial", range(40))
def test_tree_golden(lib, trial):
    from paper_2502_18890_b200 import TreeConfig, build_tree
    c = J["trees"][trial]
    t = build_tree(c["heads"], [tuple(g) for g in c["grams"]], TreeConfig(tuple(c["widths"])))
    assert t.tokens == c["tokens"]
    assert t.parent == c["parent"]
    assert t.depth == c["depth"]
    assert t.head_node_count == c["head_node_count"]
    assert [[list(p.tokens), list(p.nodes), p.origin, p.origin_index] for p in t.paths] == c["paths"]
    assert [np.nonzero(r)[0].tolist() for r in t.mask] == c["mask"]


def test_accept_commit_matches_oracle(lib):
    from paper_2502_18890_b200 import _lib as Lb
    g = np.random.default_rng(4)
    V, depth = 40, 4
    for trial in range(60):
        per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
        grams = [tuple([per_head[0][0]] + g.integers(0, V, size=3).tolist()) for _ in range(int(g.integers(0, 5)))]
        tree = OT.build_tree(per_head, grams)
        T = 1 + len(tree)
        # y biased to match the tree tokens so long paths occur
        y = g.integers(0, V, size=T)
        for r in range(T):
            kids = [i for i in range(len(tree)) if tree.parent[i] == r - 1]
            if kids and g.random() < 0.7:
                y[r] = tree.tokens[kids[int(g.integers(0, len(kids)))]]
        seed = int(g.integers(0, 1 << 62))
        n = int(g.integers(10, 1000))
        bonus = bool(trial % 5)
        pick, best_v, acc, ys, keep = OE.accept_paths(tree, y, seed, n, depth, bonus)
        rec = torch.zeros(Lb.tree_layout()["TOTAL"], dtype=torch.int32, device="cuda")
        flat = torch.tensor([t for c in per_head for t in c], dtype=torch.int32, device="cuda")
        gm = torch.tensor(grams if grams else [[0] * 4], dtype=torch.int32, device="cuda").reshape(-1)
        Lb.call("sd_tree_build", Lb.ptr(flat), Lb.host_i32([1, 3, 3, 3]), 4, Lb.ptr(gm), None, len(grams), None,
                n - 1, Lb.ptr(rec), Lb.stream())
        yt = torch.as_tensor(y.astype(np.int32), device="cuda")
        st = torch.zeros(16, dtype=torch.int64, device="cuda")
        res = torch.zeros(32, dtype=torch.int32, device="cuda")
        hist = torch.zeros(64, dtype=torch.int32, device="cuda")
        Lb.call("sd_accept_commit", Lb.ptr(rec), Lb.ptr(yt), seed, n, depth, int(bonus), Lb.ptr(st), None, None, 0,
                Lb.ptr(hist), None, Lb.ptr(res), Lb.stream())
        r = res.cpu().tolist()
        assert (r[Lb.RES_PICK], r[Lb.RES_BEST], r[Lb.RES_ACCEPTED]) == (pick, best_v, acc)
        assert r[Lb.RES_YS:Lb.RES_YS + acc] == ys
        assert r[Lb.RES_KEEP:Lb.RES_KEEP + acc] == keep
        assert r[Lb.RES_PENDING] == ys[-1]


@pytest.mark.parametrize("M", [1, 4, 41, 101, 128])
@pytest.mark.parametrize("K,N", [(4096, 6144), (4096, 4096), (512, 16384), (16384, 4096), (1024, 128)])
def test_gemm_stream_vs_fp32_reference(lib, M, K, N):
    """Weight-streaming tcgen05 GEMM (model.py:283-285, 306-309) vs a torch fp32
    reference on the same bf16 operands: fp32 split-K slices summed in order,
    and fused SiLU -> bf16; deterministic (two calls bitwise equal)."""
    import ctypes
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(M * 7 + N)
    x = torch.randn((M, K), generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn((K, N), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    wt = torch.empty((N // 128, 2, K, 64), dtype=torch.bfloat16, device=dev)
    lib.call("sd_tile_weight", lib.ptr(w), K, N, lib.ptr(wt), lib.stream())
    assert torch.equal(wt, w.reshape(K, N // 128, 2, 64).permute(1, 2, 0, 3))
    ws = torch.zeros(max(256, lib.load().sd_gemm_workspace_bytes(M, N, K)), dtype=torch.uint8, device=dev)
    tm = ctypes.create_string_buffer(128)
    lib.call("sd_make_weight_tmap", lib.ptr(wt), K, N, tm)
    want = x.float() @ w.float()
    S = lib.load().sd_gemm_splits(M, N, K, lib.GEMM_EPI_F32)
    assert S >= 1
    ys = []
    for _ in range(2):
        y = torch.full((S, M, N), float("nan"), dtype=torch.float32, device=dev)
        lib.call("sd_gemm", lib.ptr(x), M, K, tm, N, lib.GEMM_EPI_F32, lib.ptr(y), N, None, 0, lib.stream())
        acc = y[0].clone()
        for s in range(1, S):
            acc += y[s]
        ys.append(acc)
    torch.testing.assert_close(ys[0], want, rtol=1e-3, atol=1e-3)
    assert torch.equal(ys[0], ys[1])
    assert lib.load().sd_gemm_splits(M, N, K, lib.GEMM_EPI_SILU_BF16) == 1
    ysil = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    for _ in range(2):  # second call: the split-SiLU counters were left zeroed
        lib.call("sd_gemm", lib.ptr(x), M, K, tm, N, lib.GEMM_EPI_SILU_BF16, lib.ptr(ysil), N, lib.ptr(ws), ws.numel(),
                 lib.stream())
        torch.testing.assert_close(ysil.float(), torch.nn.functional.silu(want), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("S", [1, 3])
def test_norm_and_rope_sum_split_slices(lib, S):
    """sd_add_rmsnorm / sd_rope_stage consume split-K slices: same result as
    the pre-summed input (slices summed in order)."""
    dev = torch.device("cuda")
    T, d, H, Hk, dh = 5, 512, 8, 2, 64
    g = torch.Generator(device=dev)
    g.manual_seed(S)
    h0 = torch.randn((T, d), generator=g, device=dev)
    sl = torch.randn((S, T, d), generator=g, device=dev)
    gain = torch.rand(d, generator=g, device=dev) + 0.5
    tot = sl[0].clone()
    for s in range(1, S):
        tot += sl[s]
    outs = []
    for delta, splits, stride in ((tot, 1, 0), (sl, S, T * d)):
        h = h0.clone()
        x = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
        lib.call("sd_add_rmsnorm", lib.ptr(h), lib.ptr(delta), T, d, lib.ptr(gain), 1e-6, lib.ptr(x), 1, splits,
                 stride, lib.stream())
        outs.append((h, x))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    W = (H + 2 * Hk) * dh
    q = torch.randn((S, T, W), generator=g, device=dev)
    qt = q[0].clone()
    for s in range(1, S):
        qt += q[s]
    pos = torch.arange(T, dtype=torch.int32, device=dev) + 7
    inv = 10000.0 ** (-np.arange(0, dh, 2) / dh)
    ang = np.arange(64)[:, None] * inv[None]
    cs = torch.as_tensor(np.cos(ang), dtype=torch.float32, device=dev)
    sn = torch.as_tensor(np.sin(ang), dtype=torch.float32, device=dev)
    res = []
    for src, splits, stride in ((qt, 1, 0), (q, S, T * W)):
        q_rot = torch.empty((T, H, dh), dtype=torch.bfloat16, device=dev)
        kr = torch.zeros((Hk, 32, dh), dtype=torch.bfloat16, device=dev)
        kro, vv = torch.zeros_like(kr), torch.zeros_like(kr)
        lib.call("sd_rope_stage", lib.ptr(src), T, H, Hk, dh, lib.ptr(pos), lib.ptr(cs), lib.ptr(sn), 0.125,
                 lib.ptr(q_rot), 1, None, lib.ptr(kr), lib.ptr(kro), lib.ptr(vv), 1, 32 * dh, 3, None, splits, stride,
                 lib.stream())
        res.append((q_rot, kr, kro, vv))
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)


@pytest.fixture(params=["ld", "tma"])
def gemv_impl(request, monkeypatch):
    """Both weight-streaming implementations: per-lane 16-byte loads, TMA ring."""
    monkeypatch.setenv("SD_GEMV_IMPL", request.param)
    return request.param


@pytest.mark.parametrize("K,N", [(4096, 6144), (4096, 4096), (4096, 16384), (16384, 4096), (256, 512), (64, 40),
                                 (100, 8), (4096, 128256 // 16)])
def test_gemv_vs_fp32_reference(lib, K, N, gemv_impl):
    """Single-row weight streaming (draft forward projections, model.py:283-309):
    fp32 out and fused SiLU -> bf16; deterministic split-K reduction; the
    counter head is left zeroed so back-to-back calls (graph replays) work."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(K + N)
    x = torch.randn((1, K), generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn((K, N), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    ws = torch.zeros(max(256, lib.load().sd_gemv_workspace_bytes(K, N)), dtype=torch.uint8, device=dev)
    want = x.float() @ w.float()
    ys = []
    for _ in range(2):
        y = torch.full((1, N), float("nan"), device=dev)
        lib.call("sd_gemv", lib.ptr(x), K, lib.ptr(w), N, lib.GEMM_EPI_F32, lib.ptr(y), lib.ptr(ws), ws.numel(),
                 lib.stream())
        ys.append(y)
    torch.testing.assert_close(ys[0], want, rtol=1e-4, atol=1e-4)
    assert torch.equal(ys[0], ys[1])
    ysil = torch.empty((1, N), dtype=torch.bfloat16, device=dev)
    lib.call("sd_gemv", lib.ptr(x), K, lib.ptr(w), N, lib.GEMM_EPI_SILU_BF16, lib.ptr(ysil), lib.ptr(ws), ws.numel(),
             lib.stream())
    torch.testing.assert_close(ysil.float(), torch.nn.functional.silu(want), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("K,N", [(4096, 4096), (16384, 4096), (13824, 5120), (256, 512), (64, 40)])
@pytest.mark.parametrize("xdt", [torch.bfloat16, torch.float32])
def test_gemv_addnorm_vs_fp32_reference(lib, K, N, xdt, gemv_impl):
    """Projection + residual add + RMSNorm in one launch (model.py:278, 306-311):
    h += x . W, x_out = h * gain / rms(h); the row counter is left zeroed so a
    second call (graph replay) works."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(K * 7 + N)
    x = torch.randn((1, K), generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn((K, N), generator=g, device=dev) * K ** -0.5).to(torch.bfloat16)
    gain = torch.rand((N,), generator=g, device=dev) + 0.5
    h0 = torch.randn((1, N), generator=g, device=dev)
    ws = torch.zeros(lib.load().sd_gemv_workspace_bytes(K, N), dtype=torch.uint8, device=dev)
    h = h0.clone()
    for rep in range(2):
        out = torch.empty((1, N), dtype=xdt, device=dev)
        lib.call("sd_gemv_addnorm", lib.ptr(x), K, lib.ptr(w), N, lib.ptr(h), lib.ptr(gain), 1e-6, lib.ptr(out),
                 lib.dcode(xdt), lib.ptr(ws), ws.numel(), lib.stream())
        want_h = h0 + (rep + 1) * (x.float() @ w.float())
        torch.testing.assert_close(h, want_h, rtol=1e-4, atol=1e-4)
        want_x = want_h * torch.rsqrt(want_h.pow(2).mean() + 1e-6) * gain
        tol = 1e-2 if xdt == torch.bfloat16 else 1e-4
        torch.testing.assert_close(out.float(), want_x, rtol=tol, atol=tol)
    assert torch.count_nonzero(ws[:4096]) == 0  # counters left zeroed


def test_gemv_shared_workspace_across_shapes(lib, gemv_impl):
    """One zeroed workspace serves every shape (the model shares it across
    layers): a narrow split call's partials must not land in a wider call's
    arrival counters (cfg5: w2 [20480, 5120] then w1 [5120, 20480])."""
    dev = torch.device("cuda")
    shapes = [(20480, 5120), (5120, 20480), (4096, 6144), (5120, 20480)]
    need = max(lib.load().sd_gemv_workspace_bytes(K, N) for K, N in shapes)
    ws = torch.zeros(need, dtype=torch.uint8, device=dev)
    for K, N in shapes:
        x = torch.randn((1, K), device=dev).to(torch.bfloat16)
        w = (torch.randn((K, N), device=dev) * K ** -0.5).to(torch.bfloat16)
        y = torch.empty((1, N), device=dev)
        lib.call("sd_gemv", lib.ptr(x), K, lib.ptr(w), N, lib.GEMM_EPI_F32, lib.ptr(y), lib.ptr(ws), ws.numel(),
                 lib.stream())
        torch.testing.assert_close(y, x.float() @ w.float(), rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("d,H,Hk", [(4096, 32, 8), (1536, 12, 2), (5120, 40, 8)])
@pytest.mark.parametrize("normed", [False, True])
def test_gemv_rope_equals_gemv_then_rope_stage(lib, d, H, Hk, normed):
    """The draft row's QKV projection with RoPE + staging in its epilogue
    (sd_gemv_rope) equals sd_gemv(_norm) followed by sd_rope_stage bit for bit
    (same split-K reduction, same rotation arithmetic; model.py:216-232)."""
    import paper_2502_18890_b200 as sd
    dev = torch.device("cuda")
    dh = 128
    N = (H + 2 * Hk) * dh
    m = sd.TinyTransformer(sd.ModelConfig(vocab_size=256, num_layers=1, hidden_dim=d, num_heads=H, num_kv_heads=Hk,
                                          gamma=3, max_positions=4096), dtype=torch.bfloat16, init="device")
    ws = torch.zeros(lib.load().sd_gemv_workspace_bytes(d, N), dtype=torch.uint8, device=dev)
    w = (torch.randn((d, N), device=dev) * d ** -0.5).to(torch.bfloat16)
    pos = torch.tensor([1234], dtype=torch.int32, device=dev)
    x = torch.randn((1, d), device=dev).to(torch.bfloat16)
    h_in = torch.randn((1, d), device=dev)
    delta = torch.randn((1, d), device=dev)
    gain = torch.rand((d,), device=dev) + 0.5
    outs = []
    for fused in (False, True):
        q = torch.full((1, H, dh), float("nan"), dtype=torch.bfloat16, device=dev)
        k = torch.full((Hk, 1, dh), float("nan"), dtype=torch.bfloat16, device=dev)
        v = torch.full((Hk, 1, dh), float("nan"), dtype=torch.bfloat16, device=dev)
        h_out = torch.empty_like(h_in)
        if fused:
            args = ((None, lib.ptr(h_in), lib.ptr(delta), lib.ptr(gain), 1e-6, lib.ptr(h_out)) if normed
                    else (lib.ptr(x), None, None, None, 1e-6, None))
            lib.call("sd_gemv_rope", *args, d, lib.ptr(w), N, lib.ptr(pos), lib.ptr(m.rope_cos), lib.ptr(m.rope_sin),
                     m.q_scale, H, Hk, dh, lib.ptr(q), lib.ptr(k), lib.ptr(v), lib.ptr(ws), ws.numel(), lib.stream())
        else:
            y = torch.empty((1, N), device=dev)
            if normed:
                lib.call("sd_gemv_norm", lib.ptr(h_in), lib.ptr(delta), lib.ptr(gain), 1e-6, lib.ptr(h_out), d,
                         lib.ptr(w), N, lib.GEMM_EPI_F32, lib.ptr(y), lib.ptr(ws), ws.numel(), lib.stream())
            else:
                lib.call("sd_gemv", lib.ptr(x), d, lib.ptr(w), N, lib.GEMM_EPI_F32, lib.ptr(y), lib.ptr(ws), ws.numel(),
                         lib.stream())
            m.rope_stage(y, 1, pos, q, None, None, k, v, dh, 0)
        outs.append((q.clone(), k.clone(), v.clone(), h_out.clone() if normed else None))
    for a, b in zip(outs[0][:3], outs[1][:3]):
        assert torch.equal(a, b)
    if normed:
        assert torch.equal(outs[0][3], outs[1][3])


@pytest.mark.parametrize("V", [64, 5000, 151936])
@pytest.mark.parametrize("trunc", ["none", "min_p", "top_p"])
@pytest.mark.parametrize("pad", [0, 7])
def test_cluster_sampler_equals_row_sampler(lib, V, trunc, pad):
    """Engine-path sampler (8-CTA cluster per row, DSMEM reductions, top-p radix
    descent across the cluster) draws the same tokens as the single-CTA row
    sampler (selected by requesting probs_out) on fp32 logits with per-row
    window splices (engine.py:155-181, sampling.py:142-224)."""
    from paper_2502_18890_b200 import _lib as Lb
    from paper_2502_18890_b200.sampling import PenaltyWindow
    g = np.random.default_rng(V)
    W, depth = 64, 4
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    dw = PenaltyWindow(W, V, state=st)
    dw.push_many(g.integers(0, V, size=40).tolist())
    per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
    rec = torch.zeros(Lb.tree_layout()["TOTAL"], dtype=torch.int32, device="cuda")
    flat = torch.tensor([t for c in per_head for t in c], dtype=torch.int32, device="cuda")
    Lb.call("sd_tree_build", Lb.ptr(flat), Lb.host_i32([1, 3, 3, 3]), 4, None, None, 0, None, 99, Lb.ptr(rec),
            Lb.stream())
    T = 41 + pad  # rows past the tree's 41 are padding (fixed-shape verify): left untouched
    code, val = {"none": (Lb.TRUNC_NONE, 0.0), "min_p": (Lb.TRUNC_MIN_P, 0.1), "top_p": (Lb.TRUNC_TOP_P, 0.9)}[trunc]
    outs = []
    for trial in range(2):
        logits = torch.as_tensor(g.normal(scale=3.0, size=(T, V)), dtype=torch.float32, device="cuda")
        for use_row in (False, True):
            y = torch.full((T,), -1, dtype=torch.int32, device="cuda")
            probs = torch.empty((T, V), dtype=torch.float64, device="cuda") if use_row else None
            a = Lb.SampleArgs()
            a.rows, a.V, a.in_kind = T, V, Lb.IN_LOGITS_F32
            a.temperature, a.theta, a.ctrl_style = 0.9, 1.2, 0
            a.member_kind = Lb.MEMBER_TREE
            a.win_count, a.win_ring, a.state, a.window = Lb.ptr(dw.count), Lb.ptr(dw.ring), Lb.ptr(st), W
            a.tree, a.depth = Lb.ptr(rec), depth
            a.trunc_kind, a.trunc_value, a.eta_alpha = code, val, -1.0
            a.seed, a.n = trial, 100
            a.probs_out, a.token_out = Lb.ptr(probs), Lb.ptr(y)
            Lb.call("sd_sample_rows", Lb.ptr(logits), a, Lb.stream())
            outs.append(y.cpu().tolist())
        assert outs[-2] == outs[-1], (trunc, V, trial)
        assert all(0 <= t < V for t in outs[-1][:41])
        assert all(t == -1 for t in outs[-2][41:])


@pytest.mark.parametrize("d", [4096, 5120, 40, 8])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_embed_rows(lib, d, dtype):
    """Embedding gather (model.py:234-236): 16-byte bf16 loads when d % 8 == 0,
    scalar otherwise; fp32 out."""
    dev = torch.device("cuda")
    V = 1000
    E = torch.randn((V, d), device=dev).to(dtype)
    tok = torch.tensor([5, 999, 0, 5, 123], dtype=torch.int32, device=dev)
    h = torch.full((5, d), float("nan"), device=dev)
    lib.call("sd_embed", lib.ptr(tok), 5, lib.ptr(E), lib.dcode(dtype), d, lib.ptr(h), lib.stream())
    assert torch.equal(h, E[tok.long()].float())
