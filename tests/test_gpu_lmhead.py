"""Fused verification LM head (sd_lmhead_sample_stats, tcgen05) + the sampler's
scaled-input path (SD_IN_SCALED_F32), against the unfused path: fp32 GEMM of the
same bf16 operands, then the engine sampler on raw logits (engine.py:237-245,
sampling.py:98-224)."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Lb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2502_18890_b200 import _lib
    _lib.load()
    return _lib


def _tree_and_window(Lb, V, g):
    from paper_2502_18890_b200.sampling import PenaltyWindow
    W = 64
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    dw = PenaltyWindow(W, V, state=st)
    dw.push_many(g.integers(0, V, size=40).tolist())
    per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
    rec = torch.zeros(Lb.tree_layout()["TOTAL"], dtype=torch.int32, device="cuda")
    flat = torch.tensor([t for c in per_head for t in c], dtype=torch.int32, device="cuda")
    Lb.call("sd_tree_build", Lb.ptr(flat), Lb.host_i32([1, 3, 3, 3]), 4, None, None, 0, None, 99, Lb.ptr(rec),
            Lb.stream())
    return st, dw, rec, W


def _args(Lb, T, V, st, dw, rec, W, code, val, seed, ctrl=0):
    a = Lb.SampleArgs()
    a.rows, a.V, a.in_kind = T, V, Lb.IN_LOGITS_F32
    a.temperature, a.theta, a.ctrl_style = 0.9, 1.2, ctrl
    a.member_kind = Lb.MEMBER_TREE
    a.win_count, a.win_ring, a.state, a.window = Lb.ptr(dw.count), Lb.ptr(dw.ring), Lb.ptr(st), W
    a.tree, a.depth = Lb.ptr(rec), 4
    a.trunc_kind, a.trunc_value, a.eta_alpha = code, val, -1.0
    a.seed, a.n = seed, 100
    return a


@pytest.mark.parametrize("V,K", [(1000, 256), (32000, 512), (128256, 4096)])
@pytest.mark.parametrize("trunc", ["none", "min_p", "top_p"])
@pytest.mark.parametrize("pad", [0, 60])
def test_lmhead_fused_equals_unfused(Lb, V, K, trunc, pad):
    g = np.random.default_rng(V + K)
    st, dw, rec, W = _tree_and_window(Lb, V, g)
    T = 41 + pad  # rows past the tree's 41 are padding: never written, never drawn
    code, val = {"none": (Lb.TRUNC_NONE, 0.0), "min_p": (Lb.TRUNC_MIN_P, 0.1), "top_p": (Lb.TRUNC_TOP_P, 0.9)}[trunc]
    E = (torch.randn((V, K), device="cuda") * (3.0 / K ** 0.5)).to(torch.bfloat16)
    tm = ctypes.create_string_buffer(128)
    Et = torch.empty(Lb.load().sd_lmhead_tiled_bytes(V, K), dtype=torch.uint8, device="cuda")
    Lb.call("sd_tile_lmhead", Lb.ptr(E), V, K, Lb.ptr(Et), Lb.stream())
    Lb.call("sd_make_lmhead_tmap", Lb.ptr(Et), V, K, tm)
    tiles = Lb.load().sd_lmhead_tiles(V)
    assert tiles == (V + 127) // 128
    for trial in range(2):
        x = torch.randn((T, K), device="cuda").to(torch.bfloat16)
        # unfused: fp32 product of the same bf16 operands -> engine sampler
        raw = x.float() @ E.float().t()
        y_ref = torch.full((T,), -1, dtype=torch.int32, device="cuda")
        a = _args(Lb, T, V, st, dw, rec, W, code, val, trial)
        a.token_out = Lb.ptr(y_ref)
        Lb.call("sd_sample_rows", Lb.ptr(raw), a, Lb.stream())
        # the row sampler's penalised softmax (fp64) of the same raw logits
        probs = torch.empty((T, V), dtype=torch.float64, device="cuda")
        a2 = _args(Lb, T, V, st, dw, rec, W, Lb.TRUNC_NONE, 0.0, trial)
        a2.probs_out = Lb.ptr(probs)
        Lb.call("sd_sample_rows", Lb.ptr(raw), a2, Lb.stream())
        # fused
        s = torch.full((T, V), float("nan"), device="cuda")
        stats = torch.full((T, tiles, 2), float("nan"), dtype=torch.float64, device="cuda")
        y = torch.full((T,), -1, dtype=torch.int32, device="cuda")
        a3 = _args(Lb, T, V, st, dw, rec, W, code, val, trial)
        a3.token_out = Lb.ptr(y)
        Lb.call("sd_lmhead_sample_stats", Lb.ptr(x), T, K, tm, V, a3, Lb.ptr(s), Lb.ptr(stats), Lb.stream())
        a3.in_kind, a3.stats, a3.stats_tiles = Lb.IN_SCALED_F32, Lb.ptr(stats), tiles
        Lb.call("sd_sample_rows", Lb.ptr(s), a3, Lb.stream())
        torch.cuda.synchronize()
        live = 41
        assert torch.isnan(s[live:]).all() and torch.isnan(stats[live:]).all()
        sl = s[:live].double()
        # scaled logits: s - max(s) == log p - log max p of the fp64 penalised softmax
        want = torch.log(probs[:live]) - torch.log(probs[:live].max(dim=1, keepdim=True).values)
        got = sl - sl.max(dim=1, keepdim=True).values
        torch.testing.assert_close(got, want, rtol=2e-5, atol=2e-4)
        # tile statistics of the kernel's own scaled logits
        pad_v = tiles * 128 - V
        sp = torch.nn.functional.pad(sl, (0, pad_v), value=float("-inf")).view(live, tiles, 128)
        mx = sp.max(dim=2).values
        assert torch.equal(stats[:live, :, 0], mx)
        se = torch.exp(sp.float() - mx.float().unsqueeze(2)).double().sum(dim=2)
        torch.testing.assert_close(stats[:live, :, 1], se, rtol=1e-5, atol=0)
        assert all(0 <= t < V for t in y.tolist()[:live]) and all(t == -1 for t in y.tolist()[live:])
        # the draws: the tcgen05 product rounds differently from cuBLAS's (fp32
        # accumulation order), so compare with the unfused sampler on the fused
        # kernel's own raw logits (temperature 1, no penalty: s == l exactly) — the
        # scaled path must then draw the same tokens (only Z's summation order differs)
        raw_tc = torch.empty((T, V), device="cuda")
        a4 = _args(Lb, T, V, st, dw, rec, W, code, val, trial)
        a4.temperature, a4.theta, a4.member_kind = 1.0, 1.0, Lb.MEMBER_NONE
        Lb.call("sd_lmhead_sample_stats", Lb.ptr(x), T, K, tm, V, a4, Lb.ptr(raw_tc), Lb.ptr(stats), Lb.stream())
        torch.testing.assert_close(raw_tc, raw, rtol=1e-5, atol=1e-4)
        y_tc = torch.full((T,), -1, dtype=torch.int32, device="cuda")
        a5 = _args(Lb, T, V, st, dw, rec, W, code, val, trial)
        a5.token_out = Lb.ptr(y_tc)
        Lb.call("sd_sample_rows", Lb.ptr(raw_tc), a5, Lb.stream())
        assert y.tolist() == y_tc.tolist(), (V, trunc, trial)
        if trunc == "min_p":  # few, well-separated survivors: the cuBLAS path draws the same
            assert y.tolist() == y_ref.tolist(), (V, trunc, trial)


def test_lmhead_scaled_input_requires_stats(Lb):
    V = 256
    T = 4
    s = torch.zeros((T, V), device="cuda")
    y = torch.zeros((T,), dtype=torch.int32, device="cuda")
    a = Lb.SampleArgs()
    a.rows, a.V, a.in_kind = T, V, Lb.IN_SCALED_F32
    a.temperature, a.theta = 1.0, 1.0
    a.positions = None
    pos = torch.arange(T, dtype=torch.int32, device="cuda")
    a.positions = Lb.ptr(pos)
    a.token_out = Lb.ptr(y)
    with pytest.raises(Lb.LibraryError, match="tile statistics"):
        Lb.call("sd_sample_rows", Lb.ptr(s), a, Lb.stream())
