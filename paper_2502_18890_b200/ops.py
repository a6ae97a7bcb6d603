"""torch.ops.swiftdec_b200.* — the §8(b) boundary as PyTorch operators.

A thin torch.library shim over the C ABI (include/swiftdec_b200.h, loaded by
_lib): each operator takes torch tensors (device memory owned by the caller,
in-place outputs declared in the schema), resolves pointers, strides and the
current CUDA stream, and makes exactly one C-ABI call. The names follow SURVEY
§8(b)'s export list; the reference functions each replaces:

  verify_attention     model.py:238-247, 290-300 (tree rows under the ancestor mask)
  draft_attention      model.py:301-305, kvcache.py:158-165 (rank RoPE on load)
  stage_kv_rope        model.py:216-232, 276-289
  score_select_gather  kvcache.py:243-297, engine.py:128-151 (fused refresh)
  partial_admit_evict  kvcache.py:215-225, 332-354
  reconcile_rows       kvcache.py:116-127, engine.py:278-280
  ngram_update         ngram.py:35-50
  ngram_retrieve       ngram.py:52-66
  draft_topw           engine.py:207-215 (penalised per-head top-w, ties to the lower id)
  tree_build           tree.py:87-175
  verify_sample        engine.py:155-181, 237-245, sampling.py:142-224 (tree-row splice, draw)
  accept               engine.py:247-290, rng.py:23-38 (paths, uniform pick, commit)

Validation and the typed exceptions stay in the Python mirror (model.py,
kvcache.py, ngram.py); an operator raises _lib.LibraryError when the library
rejects a call. The operators are registered for CUDA tensors only: there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib as L

NS = "swiftdec_b200"
_lib = torch.library.Library(NS, "DEF")

_SCHEMAS = {
    "verify_attention": "verify_attention(Tensor q, Tensor k_rot, Tensor v, int layer, int ctx, Tensor mask_bits, "
                        "Tensor(a!) out, Tensor(b!) workspace, int kv_heads_total=0, Tensor? rows=None) -> ()",
    "draft_attention": "draft_attention(Tensor q, Tensor pk, Tensor pv, Tensor ranks, int layer, int hi, "
                       "Tensor k_self, Tensor v_self, Tensor rope_cos, Tensor rope_sin, Tensor(a!) out, "
                       "Tensor(b!) workspace, int kv_heads_total=0) -> ()",
    "stage_kv_rope": "stage_kv_rope(Tensor qkv, Tensor positions, Tensor rope_cos, Tensor rope_sin, float q_scale, "
                     "int H, int row_offset, Tensor(a!) q_rot, Tensor(b!) q_pre, Tensor(c!) k_raw, Tensor(d!) k_rot, "
                     "Tensor(e!) v, Tensor? rows=None) -> ()",
    "score_select_gather": "score_select_gather(Tensor q_sum, Tensor full_k_raw, Tensor full_v, int upto, int sink, "
                           "int budget, Tensor(a!) pk, Tensor(b!) pv, Tensor(c!) ppos, Tensor(d!) prank, "
                           "Tensor(e!) pscore, Tensor(f!) ring, Tensor(g!) freel, Tensor(h!) meta, "
                           "Tensor(i!) workspace) -> ()",
    "partial_admit_evict": "partial_admit_evict(Tensor full_k_raw, Tensor full_v, int first_pos, int count, "
                           "int evict, int protected, int sink, int budget, Tensor(a!) pk, Tensor(b!) pv, "
                           "Tensor(c!) ppos, Tensor(d!) prank, Tensor(e!) pscore, Tensor(f!) ring, Tensor(g!) freel, "
                           "Tensor(h!) meta, Tensor? result=None) -> ()",
    "reconcile_rows": "reconcile_rows(Tensor result, int base_len, Tensor(a!) k_raw, Tensor(b!) k_rot, Tensor(c!) v, "
                      "Tensor q_pre, Tensor(d!) q_sum) -> ()",
    "ngram_update": "ngram_update(Tensor(a!) table, Tensor seq, int n_tail, int n_new) -> ()",
    "ngram_retrieve": "ngram_retrieve(Tensor table, Tensor first, int k, Tensor(a!) out_grams, "
                      "Tensor(b!) out_count) -> ()",
    "draft_topw": "draft_topw(Tensor logits, Tensor? win_count, float temperature, float theta, int ctrl_style, "
                  "int[] widths, Tensor(a!) out) -> ()",
    "tree_build": "tree_build(Tensor per_head, int[] widths, int depth, Tensor grams, int n_grams, Tensor? state, "
                  "int base_pos, Tensor(a!) tree) -> ()",
    "verify_sample": "verify_sample(Tensor logits, Tensor win_count, Tensor win_ring, Tensor state, int window, "
                     "Tensor tree, int depth, float temperature, float theta, int trunc_kind, float trunc_value, "
                     "int seed, int n, Tensor(a!) token_out) -> ()",
    "accept": "accept(Tensor tree, Tensor y, int select_seed, int n, int depth, bool bonus, Tensor(a!) state, "
              "Tensor(b!) win_ring, Tensor(c!) win_count, int window, Tensor(d!) history, Tensor(e!) result, "
              "Tensor(f!)? ngram_table=None) -> ()",
}
for _s in _SCHEMAS.values():
    _lib.define(_s)

_TMAPS: dict = {}


def _tmap(kind: str, t: torch.Tensor) -> ctypes.Array:
    """128-byte TMA descriptor over a whole [L][Hk][cap][128] bf16 cache array
    (sd_make_kv_tmap / sd_make_slot_tmap), cached per (kind, pointer, shape)."""
    key = (kind, t.data_ptr(), tuple(t.shape))
    m = _TMAPS.get(key)
    if m is None:
        m = ctypes.create_string_buffer(128)
        Ln, Hk, cap, dh = t.shape
        L.call("sd_make_kv_tmap" if kind == "kv" else "sd_make_slot_tmap", L.ptr(t), Ln, Hk, cap, dh, m)
        if len(_TMAPS) > 256:
            _TMAPS.clear()
        _TMAPS[key] = m
    return m


def _tc_ok(k: torch.Tensor) -> bool:
    return k.dtype == torch.bfloat16 and k.shape[-1] == 128 and k.is_contiguous()


def _impl(name):
    def deco(fn):
        _lib.impl(name, fn, "CUDA")
        return fn
    return deco


@_impl("verify_attention")
def _verify_attention(q, k_rot, v, layer, ctx, mask_bits, out, workspace, kv_heads_total=0, rows=None):
    """q [T, H, dh] (rotated, scaled); k_rot / v [L, Hk, cap, dh] with the tree
    rows staged at [ctx, ctx + T); mask_bits [T, SD_MASK_WORDS]; out [T, H, dh]."""
    T, H, dh = q.shape
    Ln, Hk, cap, _ = k_rot.shape
    kd = L.dcode(k_rot.dtype)
    hs = cap * dh
    tk, tv = (_tmap("kv", k_rot), _tmap("kv", v)) if _tc_ok(k_rot) else (None, None)
    L.call("sd_attention", L.ptr(q), L.dcode(q.dtype), T, H, Hk, dh, 0, L.ptr(k_rot[layer]), L.ptr(v[layer]), kd,
           hs, ctx, None, None, None, L.ptr(k_rot[layer, :, ctx:]), L.ptr(v[layer, :, ctx:]), hs, L.ptr(mask_bits),
           mask_bits.shape[-1], L.ptr(rows), None, tk, tv, layer, kv_heads_total, L.ptr(out), L.dcode(out.dtype),
           L.ptr(workspace), workspace.numel(), L.stream())


@_impl("draft_attention")
def _draft_attention(q, pk, pv, ranks, layer, hi, k_self, v_self, rope_cos, rope_sin, out, workspace,
                     kv_heads_total=0):
    """q [1, H, dh] rotated at the draft rank; pk / pv [L, Hk, cap, dh] partial
    slots (pre-rotation K); ranks [L, cap] (< 0: hole); k_self / v_self [Hk, dh]
    the pending row (rotated); out [1, H, dh]."""
    _, H, dh = q.shape
    Ln, Hk, cap, _ = pk.shape
    kd = L.dcode(pk.dtype)
    tk, tv = (_tmap("slot", pk), _tmap("slot", pv)) if _tc_ok(pk) else (None, None)
    L.call("sd_attention", L.ptr(q), L.dcode(q.dtype), 1, H, Hk, dh, 1, L.ptr(pk[layer]), L.ptr(pv[layer]), kd,
           cap * dh, hi, L.ptr(ranks[layer]), L.ptr(rope_cos), L.ptr(rope_sin), L.ptr(k_self), L.ptr(v_self),
           k_self.stride(0), None, 0, None, None, tk, tv, layer, kv_heads_total, L.ptr(out), L.dcode(out.dtype),
           L.ptr(workspace), workspace.numel(), L.stream())


@_impl("stage_kv_rope")
def _stage_kv_rope(qkv, positions, rope_cos, rope_sin, q_scale, H, row_offset, q_rot, q_pre, k_raw, k_rot, v,
                   rows=None):
    """qkv [T, (H + 2 Hk) dh] fp32 (or [S, T, N] split-K slices); k_raw / k_rot /
    v: one layer's cache [Hk, cap, dh], rows written at row_offset + t."""
    Hk, cap, dh = k_rot.shape
    T = qkv.shape[-2]
    S, sstride = (qkv.shape[0], qkv.shape[1] * qkv.shape[2]) if qkv.dim() == 3 else (1, 0)
    L.call("sd_rope_stage", L.ptr(qkv), T, H, Hk, dh, L.ptr(positions), L.ptr(rope_cos), L.ptr(rope_sin), q_scale,
           L.ptr(q_rot), L.dcode(q_rot.dtype), L.ptr(q_pre), L.ptr(k_raw), L.ptr(k_rot), L.ptr(v),
           L.dcode(k_rot.dtype), cap * dh, row_offset, L.ptr(rows), S, sstride, L.stream())


def _slot_args(ppos, prank, pscore, ring, freel, meta):
    return (ppos.shape[-1], L.ptr(ppos), L.ptr(prank), L.ptr(pscore), L.ptr(ring), L.ptr(freel), L.ptr(meta))


@_impl("score_select_gather")
def _score_select_gather(q_sum, full_k_raw, full_v, upto, sink, budget, pk, pv, ppos, prank, pscore, ring, freel,
                         meta, workspace):
    """q_sum [L, H, dh] fp32; full_k_raw / full_v [L, Hk, cap, dh]; pk / pv
    [L, Hk, slot_cap, dh]; slot arrays as PartialCache (kvcache.py)."""
    Ln, H, dh = q_sum.shape
    _, Hk, fcap, _ = full_k_raw.shape
    _, _, scap, _ = pk.shape
    L.call("sd_partial_refresh", L.ptr(q_sum), None, Ln, H, Hk, dh, upto, sink, budget, L.ptr(full_k_raw),
           L.ptr(full_v), L.dcode(pk.dtype), Hk * fcap * dh, fcap * dh, L.ptr(pk), L.ptr(pv), Hk * scap * dh,
           scap * dh, *_slot_args(ppos, prank, pscore, ring, freel, meta), L.ptr(workspace), workspace.numel(),
           L.stream())


@_impl("partial_admit_evict")
def _partial_admit_evict(full_k_raw, full_v, first_pos, count, evict, protected, sink, budget, pk, pv, ppos, prank,
                         pscore, ring, freel, meta, result=None):
    Ln, Hk, fcap, dh = full_k_raw.shape
    _, _, scap, _ = pk.shape
    L.call("sd_partial_step", Ln, L.ptr(result), count, first_pos, evict, protected, sink, budget, Hk, dh,
           L.ptr(full_k_raw), L.ptr(full_v), L.dcode(pk.dtype), Hk * fcap * dh, fcap * dh, L.ptr(pk), L.ptr(pv),
           Hk * scap * dh, scap * dh, *_slot_args(ppos, prank, pscore, ring, freel, meta), L.stream())


@_impl("reconcile_rows")
def _reconcile_rows(result, base_len, k_raw, k_rot, v, q_pre, q_sum):
    """k_raw / k_rot / v [L, Hk, cap, dh]; q_pre [L, T, H, dh]; q_sum [L, H, dh]."""
    Ln, Hk, cap, dh = k_rot.shape
    _, T, H, _ = q_pre.shape
    L.call("sd_reconcile", Ln, L.ptr(result), base_len, L.ptr(k_raw), L.ptr(k_rot), L.ptr(v), L.dcode(k_rot.dtype),
           Hk * cap * dh, cap * dh, Hk, dh, L.ptr(q_pre), T, H, L.ptr(q_sum), L.stream())


@_impl("ngram_update")
def _ngram_update(table, seq, n_tail, n_new):
    L.call("sd_ngram_update", L.ptr(table), L.ptr(seq), n_tail, n_new, L.stream())


@_impl("ngram_retrieve")
def _ngram_retrieve(table, first, k, out_grams, out_count):
    L.call("sd_ngram_retrieve", L.ptr(table), L.ptr(first), k, L.ptr(out_grams), L.ptr(out_count), L.stream())


@_impl("draft_topw")
def _draft_topw(logits, win_count, temperature, theta, ctrl_style, widths, out):
    """logits [heads, V] fp32 -> out: concatenated candidates, head k gets widths[k]."""
    heads, V = logits.shape
    L.call("sd_draft_topw", L.ptr(logits), heads, V, L.ptr(win_count), temperature, theta, ctrl_style,
           L.host_i32(widths), L.ptr(out), L.stream())


@_impl("tree_build")
def _tree_build(per_head, widths, depth, grams, n_grams, state, base_pos, tree):
    """per_head: concatenated candidates; grams [n_grams, depth]; tree: the
    device tree record (sd_tree_layout)."""
    L.call("sd_tree_build", L.ptr(per_head), L.host_i32(widths), depth, L.ptr(grams), None, n_grams, L.ptr(state),
           base_pos, L.ptr(tree), L.stream())


@_impl("verify_sample")
def _verify_sample(logits, win_count, win_ring, state, window, tree, depth, temperature, theta, trunc_kind,
                   trunc_value, seed, n, token_out):
    """logits [rows, V] fp32 of the tree rows; each row's window is the committed
    window spliced with its branch (member kind TREE); one draw per row at the
    tree-derived position key (row 0 -> n, node -> n + depth + 1)."""
    rows, V = logits.shape
    a = L.SampleArgs()
    a.rows, a.V, a.in_kind = rows, V, L.IN_LOGITS_F32
    a.temperature, a.theta, a.ctrl_style = temperature, theta, 0
    a.trunc_kind, a.trunc_value, a.eta_alpha = trunc_kind, trunc_value, -1.0
    a.seed = seed & ((1 << 64) - 1)
    a.member_kind = L.MEMBER_TREE
    a.win_count, a.win_ring, a.state, a.window = L.ptr(win_count), L.ptr(win_ring), L.ptr(state), window
    a.tree, a.depth = L.ptr(tree), depth
    a.positions, a.n = None, n
    a.token_out = L.ptr(token_out)
    L.call("sd_sample_rows", L.ptr(logits), a, L.stream())


@_impl("accept")
def _accept(tree, y, select_seed, n, depth, bonus, state, win_ring, win_count, window, history, result,
            ngram_table=None):
    L.call("sd_accept_commit", L.ptr(tree), L.ptr(y), select_seed & ((1 << 64) - 1), n, depth, int(bonus),
           L.ptr(state), L.ptr(win_ring), L.ptr(win_count), window, L.ptr(history), L.ptr(ngram_table),
           L.ptr(result), L.stream())


def schemas() -> dict:
    """Operator name -> schema string (for the C-ABI / boundary tests)."""
    return dict(_SCHEMAS)
