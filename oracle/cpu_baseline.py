"""CPU baseline of the decode step, timed with the oracle port (bench only).

The reference (swiftdec) is pure Python/numpy; there is nothing to compile,
so the CPU arm is the oracle restatement of the same algorithm (kind "port").
At LLaMA-8B shapes one reference step takes tens of minutes,
so the baseline is a BOUNDED sample composed from full-shape pieces:

  per step = L x [one verification layer (T rows over a ctx-long cache)
                  + one draft layer (1 row over the B-entry partial cache)]
             + LM head (T + gamma + 1 rows; timed on a 1/`vocab_div` vocab
               slice and scaled) + penalised sampling of T rows over V
             + n-gram retrieval + tree build + acceptance.

Each piece runs the oracle code at the bench workload's real dims. numpy uses
all host cores for GEMMs (BLAS); einsum-based attention is single-threaded.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import engine as OE
from . import kvcache as OK
from . import model as OM
from . import ngram as ON
from . import sampling as OS
from . import tree as OT


def _timed(fn, reps=1):
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def compose_step(d, L, H, Hk, V, ctx, budget, widths=(1, 3, 3, 3), k=20, tree_rows=41, vocab_div=16,
                 accepted=4.0, seed=0):
    """Seconds per decode step on host cores, composed from full-shape pieces."""
    g = np.random.default_rng(seed)
    depth = len(widths)
    cfg1 = OM.ModelConfig(vocab_size=1024, num_layers=1, hidden_dim=d, num_heads=H, num_kv_heads=Hk, gamma=depth - 1,
                          max_positions=ctx + 4096)
    t_build0 = time.perf_counter()
    model = OM.TinyTransformer(cfg1)
    dh = d // H
    # verification layer: T rows over a synthetic ctx-long full cache
    full = OK.FullCache(1, Hk, dh, cap=ctx + tree_rows + 8)
    full.k_raw[0, :ctx] = g.standard_normal((ctx, Hk, dh))
    full.k_rot[0, :ctx] = full.k_raw[0, :ctx]
    full.v[0, :ctx] = g.standard_normal((ctx, Hk, dh))
    full.positions = list(range(ctx))
    per_head = [[int(x) for x in g.choice(1024, w, replace=False)] for w in widths]
    grams = [tuple([per_head[0][0]] + g.integers(0, 1024, size=depth - 1).tolist()) for _ in range(k)]
    tree = OT.build_tree(per_head, grams)
    rows = min(tree_rows, 1 + len(tree))
    mask = np.zeros((rows, ctx + rows), dtype=bool)
    mask[:, : ctx + 1] = True
    mask[1:, ctx + 1:] = tree.mask[: rows - 1, : rows - 1]
    toks = [1] + tree.tokens[: rows - 1]
    pos = [ctx] + [ctx + 1 + dd for dd in tree.depth[: rows - 1]]
    setup = time.perf_counter() - t_build0

    def verify_layer():
        full.truncate(ctx)
        model.forward(toks, pos, full, mask, heads_needed=1)

    t_verify = _timed(verify_layer)
    # draft layer: 1 row over the budget-sized partial cache view
    ks = [g.standard_normal((budget, Hk, dh))]
    vs = [g.standard_normal((budget, Hk, dh))]
    buf = model.buffer_from_view(ks, vs)

    def draft_layer():
        b = model.buffer_from_view(ks, vs)
        model.forward([1], [budget], b, heads_needed=1)

    t_draft = _timed(draft_layer)
    del buf
    # LM head on a vocab slice, scaled
    Vs = max(1, V // vocab_div)
    E = g.standard_normal((Vs, d)) * 0.3
    h = g.standard_normal((rows + depth, d))
    t_lm = _timed(lambda: h @ E.T) * (V / Vs)
    # penalised sampling over T x V (min-p 0.1 profile)
    logits = g.standard_normal((rows, V)) * 3.0
    win = OS.PenaltyWindow(1024, V)
    for t in g.integers(0, V, size=1024):
        win.push(int(t))
    smp = OS.SamplerConfig()

    def sample_rows():
        masks = OS.node_masks(win, tree.tokens[: rows - 1], tree.parent[: rows - 1], depth)
        dists = OS.penalized_probs_masked(logits, masks, smp)
        for r in range(rows):
            OS.sample_at(OS.truncate(dists[r], smp.truncation), 1000 + r, 0)

    t_sample = _timed(sample_rows)
    # draft top-w over gamma+1 heads
    hl = g.standard_normal((depth, V))
    t_topw = _timed(lambda: [np.argsort(-OS.penalized_probs_masked(hl[i], win.member_mask(), smp), kind="stable")
                             for i in range(depth)])
    # n-gram + tree + accept
    tab = ON.NGramTable(n=depth)
    seq = g.integers(0, 64, size=4000).tolist()
    tab.update(seq, [])
    y = g.integers(0, 1024, size=1 + len(tree))

    def misc():
        tab.retrieve(seq[0], k)
        t2 = OT.build_tree(per_head, grams)
        OE.accept_paths(t2, y, 7, 100, depth, True)

    t_misc = _timed(misc, reps=5)
    per_step = L * (t_verify + t_draft) + t_lm + t_sample + t_topw + t_misc
    parts = {"verify_layer_s": t_verify, "draft_layer_s": t_draft, "lm_head_s": t_lm, "sample_s": t_sample,
             "draft_topw_s": t_topw, "ngram_tree_accept_s": t_misc, "setup_s": setup}
    return per_step, accepted / per_step, parts


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
