"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json (integers, small lists) and
tests/golden/golden.npz (float arrays). These fixtures travel to the GPU box;
nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from swiftdec import engine as E  # noqa: E402
from swiftdec import kvcache as KV  # noqa: E402
from swiftdec import model as M  # noqa: E402
from swiftdec import ngram as NG  # noqa: E402
from swiftdec import rng as R  # noqa: E402
from swiftdec import sampling as S  # noqa: E402
from swiftdec import tree as TR  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
J: dict = {}
A: dict = {}


def rng_vectors():
    J["mix"] = [[s, c, R.mix(s, c)] for s, c in [(0, 0), (7, 1), (123, 456), (2**64 - 1, 5), (3, 2**40)]]
    J["uniform_at"] = [[s, c, R.uniform_at(s, c)] for s, c in [(0, 0), (3, 4096), (9, 77), (11, 100000)]]
    J["derive_seed"] = [[s, t, R.derive_seed(s, t)] for s, t in [(0, "branch-select"), (0, "prompt"), (5, "a")]]
    J["prompt_128256"] = [R.mix(R.derive_seed(0, "prompt"), i) % 128256 for i in range(32)]


def sampling_vectors():
    g = np.random.default_rng(1234)
    cases = []
    for trial in range(24):
        V = int(g.integers(16, 300))
        logits = g.normal(scale=3.0, size=V)
        if trial % 5 == 0:
            logits[g.integers(0, V, size=3)] = logits.max()  # exact ties
        members = g.random(V) < 0.2
        t = float(g.choice([0.7, 1.0, 1.3]))
        theta = float(g.choice([1.0, 1.15, 1.2, 1.5]))
        ctrl = bool(trial % 7 == 3)
        cfg = S.SamplerConfig(temperature=t, theta=theta, window=64, ctrl_style=ctrl)
        probs = S.penalized_probs_masked(logits, members, cfg)
        rules = [S.Truncation.min_p(0.1), S.Truncation.top_p(0.9), S.Truncation.eta(0.02),
                 S.Truncation.top_p(0.5), S.Truncation.min_p(0.5)]
        draws = {}
        for ri, rule in enumerate(rules):
            d = S.truncate(probs, rule)
            A[f"samp{trial}_trunc{ri}"] = d
            draws[ri] = [S.sample_at(d, pos, seed) for pos, seed in [(0, 0), (5, 1), (777, 3), (4096, 0)]]
        A[f"samp{trial}_logits"] = logits
        A[f"samp{trial}_members"] = members
        A[f"samp{trial}_probs"] = probs
        cases.append({"V": V, "t": t, "theta": theta, "ctrl": ctrl, "draws": draws})
    J["sampling"] = cases
    # shrunk masks / windows
    toks = g.integers(0, 16, size=40).tolist()
    w = S.PenaltyWindow(8, 16)
    for tk in toks:
        w.push(tk)
    J["shrunk"] = {"tokens": toks, "cap": 8, "V": 16,
                   "masks": [np.nonzero(m)[0].tolist() for m in w.shrunk_masks(5)]}


def tree_vectors():
    g = np.random.default_rng(7)
    out = []
    for trial in range(40):
        widths = [int(x) for x in g.integers(1, 4, size=int(g.integers(1, 5)))]
        heads = [[10 * k + i + int(g.integers(0, 3)) * 100 for i in range(w)] for k, w in enumerate(widths)]
        grams = []
        if trial % 3 != 0:
            for _ in range(int(g.integers(1, 8))):
                tail = [int(x) for x in g.integers(0, 3, size=len(widths) - 1)]
                # bias towards merging with head tokens
                tail = [heads[k + 1][t % len(heads[k + 1])] if g.random() < 0.5 else 999 + t
                        for k, t in enumerate(tail)]
                grams.append(tuple([heads[0][0]] + tail))
            if grams and g.random() < 0.5:
                grams.append(grams[0])
        tree = TR.build_tree(heads, grams, TR.TreeConfig(tuple(widths)))
        out.append({
            "widths": widths, "heads": heads, "grams": [list(x) for x in grams],
            "tokens": tree.tokens, "parent": tree.parent, "depth": tree.depth,
            "paths": [[list(p.tokens), list(p.nodes), p.origin, p.origin_index] for p in tree.paths],
            "head_node_count": tree.head_node_count,
            "mask": [np.nonzero(r)[0].tolist() for r in tree.mask],
        })
    J["trees"] = out


def ngram_vectors():
    g = np.random.default_rng(11)
    out = []
    for trial in range(6):
        n = int(g.integers(2, 5))
        tab = NG.NGramTable(n=n, k_max=64)
        seq: list[int] = []
        ops = []
        length = 3000 if trial == 0 else int(g.integers(50, 400))
        while len(seq) < length:
            chunk = g.integers(0, 6, size=int(g.integers(1, 5))).tolist()
            tail = seq[-(n - 1):] if n > 1 else []
            tab.update(chunk, tail)
            seq.extend(chunk)
            ops.append(chunk)
        retr = {str(f): [list(x) for x in tab.retrieve(f, 20)] for f in range(6)}
        freqs = [[list(gm), tab.frequency(gm)] for gm in sorted(tab._freq)[:50]]
        out.append({"n": n, "ops": ops, "retrieve": retr, "freqs": freqs, "size": len(tab)})
    J["ngram"] = out


def kvcache_vectors():
    g = np.random.default_rng(5)
    sc = []
    for gs in (1, 2, 4, 8):
        q = g.normal(size=(3 * gs, 5))
        keys = g.normal(size=(9, 3, 5))
        A[f"imp_q{gs}"], A[f"imp_k{gs}"] = q, keys
        A[f"imp_s{gs}"] = KV.importance_scores(q, keys, gs)
        sc.append(gs)
    J["imp_groups"] = sc
    sel = []
    for trial in range(10):
        L, n, sink, budget = 2, int(g.integers(12, 60)), int(g.integers(1, 5)), 0
        budget = int(g.integers(sink + 2, n + 1))
        cache = KV.FullCache(L, 1, 2)
        cache.reserve(n)
        for pos in range(n):
            for layer in range(L):
                k = g.normal(size=(1, 2))
                cache.stage(layer, pos - len(cache), k, k, np.full((1, 2), float(pos)))
            cache.commit_rows([pos])
        scores = np.round(g.normal(size=(L, n - sink)), 1)  # rounding creates ties
        part = KV.prefill_partial(cache, sink, budget, scores)
        A[f"sel{trial}_scores"] = scores
        sel.append({"n": n, "sink": sink, "budget": budget, "positions": part.positions})
    J["select"] = sel


def model_vectors():
    cfgs = {
        "gqa": M.ModelConfig(vocab_size=64, num_layers=2, hidden_dim=32, num_heads=4, num_kv_heads=2, gamma=3, init_seed=2),
        "mha": M.ModelConfig(vocab_size=48, num_layers=2, hidden_dim=32, num_heads=4, num_kv_heads=4, gamma=2, init_seed=5),
        "g4": M.ModelConfig(vocab_size=80, num_layers=2, hidden_dim=64, num_heads=8, num_kv_heads=2, gamma=3, init_seed=9),
    }
    meta = {}
    for name, c in cfgs.items():
        model = M.TinyTransformer(c)
        prefix = [3, 11, 7, 29, 40, 8, 1, 2, 5]
        cache = model.new_cache()
        r = model.forward(M.ForwardRequest(tokens=prefix, positions=list(range(len(prefix))), cache=cache))
        A[f"m_{name}_prefill_b"], A[f"m_{name}_prefill_q"] = r.bundles, r.queries
        heads = [[4, 9][: 1], [13, 21], [30, 31], [1, 2]][: c.gamma + 1]
        grams = [(heads[0][0],) + tuple(10 + i for i in range(c.gamma))]
        tree = TR.build_tree(heads, grams)
        ctx = len(prefix)
        rows = len(tree)
        mask = np.zeros((rows, ctx + rows), dtype=bool)
        mask[:, :ctx] = True
        for i in range(rows):
            mask[i, ctx:ctx + rows] = tree.mask[i]
        r2 = model.forward(M.ForwardRequest(tokens=tree.tokens, positions=[ctx + d for d in tree.depth],
                                            cache=cache, attention_mask=mask, heads_needed=1))
        A[f"m_{name}_tree_b"] = r2.bundles[:, 0]
        A[f"m_{name}_tree_q"] = r2.queries
        meta[name] = {"cfg": c.__dict__, "prefix": prefix, "tree_tokens": tree.tokens,
                      "tree_parent": tree.parent, "tree_depth": tree.depth}
    J["model"] = meta


def engine_vectors():
    runs = []

    def tiny(seed, kv, vocab, hidden=32, heads=4, layers=2):
        return M.TinyTransformer(M.ModelConfig(vocab_size=vocab, num_layers=layers, hidden_dim=hidden,
                                               num_heads=heads, num_kv_heads=kv, gamma=3, init_seed=seed))

    specs = [
        ("evict_minp", dict(seed=2, kv=2, vocab=64), [int(x) for x in (np.arange(24) * 5) % 64],
         dict(target_length=200, sink_size=4, budget=16, widths=(1, 2, 2, 2), k=4,
              sampler=dict(seed=11, theta=1.2, window=32, kind="min_p", value=0.1), seed=3)),
        ("short_prompt", dict(seed=7, kv=2, vocab=32), [1, 2, 3, 4],
         dict(target_length=120, sink_size=2, budget=64, widths=(1, 2, 2, 2), k=4,
              sampler=dict(seed=13, theta=1.0, window=0, kind="min_p", value=0.2), seed=3)),
        ("topp_nobonus", dict(seed=4, kv=1, vocab=40), list(range(3, 20)),
         dict(target_length=100, sink_size=2, budget=10, widths=(1, 3, 2, 2), k=6, bonus=False,
              sampler=dict(seed=4, theta=1.15, window=16, kind="top_p", value=0.8), seed=9)),
        ("eta_greedyish", dict(seed=6, kv=2, vocab=50), [5, 9, 1, 4, 7, 2, 8, 8, 3],
         dict(target_length=120, sink_size=2, budget=12, widths=(1, 3, 3, 3), k=20,
              sampler=dict(seed=2, theta=1.3, window=8, kind="eta", value=0.02, temperature=0.8), seed=1)),
        ("greedy_cfg1like", dict(seed=0, kv=2, vocab=256, hidden=64, heads=8), None,
         dict(target_length=160, sink_size=8, budget=40, widths=(1, 3, 3, 3), k=20,
              sampler=dict(seed=0, theta=1.2, window=1024, kind="min_p", value=1.0), seed=0)),
    ]
    for name, mk, prompt, ek in specs:
        model = tiny(mk["seed"], mk["kv"], mk["vocab"], mk.get("hidden", 32), mk.get("heads", 4))
        if prompt is None:
            prompt = [R.mix(R.derive_seed(0, "prompt"), i) % mk["vocab"] for i in range(48)]
        sp = dict(ek["sampler"])
        smp = S.SamplerConfig(temperature=sp.get("temperature", 1.0), theta=sp["theta"], window=sp["window"],
                              truncation=S.Truncation(sp["kind"], sp["value"]), seed=sp["seed"])
        ecfg = E.EngineConfig(target_length=ek["target_length"], sink_size=ek["sink_size"], budget=ek["budget"],
                              tree=TR.TreeConfig(ek["widths"]), k=ek["k"], sampler=smp, seed=ek["seed"],
                              bonus=ek.get("bonus", True))
        sess = E.prefill(model, prompt, ecfg)
        while not sess.done:
            sess.step()
        ar = E.generate_ar(model, prompt, E.EngineConfig(**{**ecfg.__dict__, "target_length": len(sess.emitted)}))
        runs.append({
            "name": name, "model": {**mk}, "prompt": prompt, "engine": {**ek, "widths": list(ek["widths"])},
            "emitted": sess.emitted, "ar": ar,
            "records": [[r.accepted, r.ngram_accepted, r.origin, r.matched, r.tokens, r.refreshed,
                         r.draft_ctx, r.verify_ctx, r.verify_rows, r.path_index] for r in sess.records],
            "final_partial_positions": sess.partial.positions,
            "final_mark": sess.partial.mark,
        })
    J["engine"] = runs


if __name__ == "__main__":
    rng_vectors()
    sampling_vectors()
    tree_vectors()
    ngram_vectors()
    kvcache_vectors()
    model_vectors()
    engine_vectors()
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(J, fh, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **A)
    print("wrote", len(J), "json groups,", len(A), "arrays")
