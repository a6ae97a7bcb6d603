"""Reference arm of bench.py: the UNMODIFIED reference (swiftdec, pure
Python/numpy fp64) timed on the host cores.

The package is imported from `baseline/_ref` (pip-installed from
/root/reference), else from /root/reference/pkg/src when
that tree exists; nothing here is product code and nothing in the product
imports it.

cfg1 (tiny model) runs the reference's own `Session.step()` end to end:
prefill, W warm-up steps, K timed steps, tokens/s = emitted / wall time.

cfgs 2-5 cannot run end to end on a CPU (one LLaMA-8B-shape iteration at
ctx 54K is ~10 min), so one "step" of this arm is a bounded
sample of the iteration, composed from the reference's own functions timed at
the config's full shapes (a ONE-layer model of the config's dims, the
reference initialiser, a synthetic ctx-long cache):

  verify  = L x (scratch copy + T x layer row) + T x LM-head row, from
            `TinyTransformer.forward` with a masked 1-row and 2-row request
            (rows are processed strictly one at a time, model.py:263-311, so
            the per-row increment composes exactly)
  draft   = `forward` of 1 row over the partial cache's `draft_view` with all
            gamma+1 heads, + (L-1) more layers
  cache   = L x (`PartialCache.admit` + `draft_view` + `FullCache.reconcile`)
  sample  = `_node_masks` + `penalized_probs_masked` + `truncate` +
            `sample_at` over T x V; draft top-w = penalised probs + stable argsort
  misc    = `NGramTable.update/retrieve` + `build_tree`
  refresh = L x (`importance_scores` + `prefill_partial`) amortised over the
            B - S + 1 tokens between refreshes (timed once per run)

The 1-row forward, the LM-head row and the draft-head chain are timed once
per run; every sample re-times the 2-row verify forward, the draft forward,
cache maintenance, sampling, top-w and n-gram/tree work (~5 s at cfg3).

The line says `composed: true` and gives the parts; `ms_per_step` is the
composed iteration time, not the wall time of a sample (`sample_wall_s`).
"""

from __future__ import annotations

import os
import statistics
import sys
import time
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def import_reference():
    """(swiftdec module, where it came from) or (None, why)."""
    for path in (os.path.join(HERE, "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "swiftdec")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import swiftdec
            return swiftdec, path
    return None, "swiftdec not installed in baseline/_ref and /root/reference absent"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _t(fn):
    t0 = time.perf_counter()
    r = fn()
    return time.perf_counter() - t0, r


# ------------------------------------------------------------------ cfg1 --
def run_session(c, steps, warmup):
    """The reference Session end to end (cfg1 shape): prefill, warm-up steps,
    timed steps. Returns (tokens/s, details)."""
    import swiftdec as S
    from swiftdec.rng import derive_seed, mix
    mcfg = S.ModelConfig(vocab_size=c["V"], num_layers=c["L"], hidden_dim=c["d"], num_heads=c["H"],
                         num_kv_heads=c["Hk"], gamma=3, max_positions=c["prefix"] + c["gen"] + 64, init_seed=0)
    model = S.TinyTransformer(mcfg)
    seed = derive_seed(0, "prompt")
    prompt = [mix(seed, i) % c["V"] for i in range(c["prefix"])]
    trunc = S.Truncation.min_p(c["trunc"][1]) if c["trunc"][0] == "min_p" else S.Truncation.top_p(c["trunc"][1])
    ecfg = S.EngineConfig(target_length=c["gen"], sink_size=c["S"], budget=c["B"],
                          tree=S.TreeConfig((1, 3, 3, 3)), k=20,
                          sampler=S.SamplerConfig(theta=c["theta"], window=1024, truncation=trunc))
    tp, sess = _t(lambda: S.Session(model, prompt, ecfg))
    for _ in range(warmup):
        sess.step()
    n0 = len(sess.emitted)
    t0 = time.perf_counter()
    for _ in range(steps):
        if len(sess.emitted) >= ecfg.target_length:
            break
        sess.step()
    wall = time.perf_counter() - t0
    toks = len(sess.emitted) - n0
    recs = sess.records[-steps:]
    return toks / wall, {"wall_s": wall, "tokens": toks, "prefill_s": tp,
                         "alpha": statistics.mean(r.accepted for r in recs) / 4.0,
                         "mean_verify_rows": statistics.mean(r.verify_rows for r in recs)}


# ------------------------------------------------------------- cfg2..5 --
class Composer:
    """Full-shape pieces of one reference iteration (see module docstring)."""

    def __init__(self, c, ctx, rows=41, seed=0):
        import swiftdec as S
        from swiftdec import kvcache as K
        self.S, self.K = S, K
        self.c, self.ctx, self.rows = c, ctx, rows
        g = np.random.default_rng(seed)
        self.g = g
        d, H, Hk = c["d"], c["H"], c["Hk"]
        dh = d // H
        self.mcfg = S.ModelConfig(vocab_size=c["V"], num_layers=1, hidden_dim=d, num_heads=H, num_kv_heads=Hk,
                                  gamma=3, max_positions=ctx + 4096, init_seed=0)
        t0 = time.perf_counter()
        self.model = S.TinyTransformer(self.mcfg)  # the reference initialiser, one layer of the config's dims
        full = self.model.new_cache()
        full.reserve(ctx + rows + 8)
        la = full._layers[0]
        la.k_raw[:ctx] = g.standard_normal((ctx, Hk, dh))
        la.k_rot[:ctx] = self.model.rope_rows(la.k_raw[:ctx], np.arange(ctx))
        la.v[:ctx] = g.standard_normal((ctx, Hk, dh))
        full.commit_rows(list(range(ctx)))
        self.full = full
        self.q_sum = g.standard_normal((H, dh))
        self.scores = K.importance_scores(self.q_sum, full.raw_keys(0, ctx)[c["S"]:], H // Hk)[None]
        self.partial = K.prefill_partial(full, c["S"], c["B"], self.scores, upto=ctx)
        V = c["V"]
        self.window = S.PenaltyWindow(1024, V)
        for t in g.integers(0, V, size=1024):
            self.window.push(int(t))
        trunc = S.Truncation.min_p(c["trunc"][1]) if c["trunc"][0] == "min_p" else S.Truncation.top_p(c["trunc"][1])
        self.smp = S.SamplerConfig(theta=c["theta"], window=1024, truncation=trunc)
        self.per_head = [[int(x) for x in g.choice(V, w, replace=False)] for w in (1, 3, 3, 3)]
        self.ngrams = S.NGramTable(n=4, k_max=64)
        hist = g.integers(0, 64, size=4000).tolist()
        self.ngrams.update(hist, [])
        self.tree = S.build_tree(self.per_head, [], S.TreeConfig((1, 3, 3, 3)))
        self.setup_s = time.perf_counter() - t0
        self.refresh = None

    def _verify_forward(self, nrows):
        """Reference masked forward of the root + (nrows-1) depth-chain nodes
        over the ctx-long cache, one layer, heads_needed=1 (engine.py:226-236)."""
        S, ctx = self.S, self.ctx
        self.full.truncate(ctx)
        mask = np.zeros((nrows, ctx + nrows), dtype=bool)
        mask[:, :ctx] = True
        for r in range(nrows):
            mask[r, ctx:ctx + r + 1] = True  # chain: every earlier row is an ancestor
        req = S.ForwardRequest(tokens=[1 + r for r in range(nrows)], positions=[ctx + r for r in range(nrows)],
                               cache=self.full, attention_mask=mask, heads_needed=1)
        t, _ = _t(lambda: self.model.forward(req))
        self.full.truncate(ctx)
        return t

    def time_refresh(self):
        """importance_scores + prefill_partial for one layer at ctx (kvcache.py:243-297)."""
        K, c, ctx = self.K, self.c, self.ctx
        ts, sc = _t(lambda: K.importance_scores(self.q_sum, self.full.raw_keys(0, ctx)[c["S"]:], c["H"] // c["Hk"]))
        tp, _ = _t(lambda: K.prefill_partial(self.full, c["S"], c["B"], sc[None], upto=ctx))
        self.refresh = (ts, tp)

    def sample(self, accepted=4.0):
        """One composed iteration; returns (seconds per iteration, parts)."""
        S, K, c, ctx, T = self.S, self.K, self.c, self.ctx, self.rows
        from swiftdec.sampling import penalized_probs_masked
        L, V = c["L"], c["V"]
        h0 = self.g.standard_normal(c["d"])
        embed = self.model.params["embed"]
        heads = [self.model.params[f"head{i + 1}"] for i in range(3)]
        if self.refresh is None:  # once per run: refresh pieces, 1-row forward, head chains
            self.time_refresh()
            self._verify_forward(2)  # warm: first-touch of the scratch blocks
            self.t1 = min(self._verify_forward(1) for _ in range(2))
            self.t_lm, _ = _t(lambda: S.chained_draft_logits(h0, [], embed))
            self.t_h, _ = _t(lambda: S.chained_draft_logits(h0, heads, embed))
        t1, t_lm, t_h = self.t1, self.t_lm, self.t_h
        t2 = self._verify_forward(2)
        row = max(t2 - t1, 1e-9)            # one more row: layer row + LM-head row
        layer_row = max(row - t_lm, 0.0)
        scratch = max(t1 - row, 0.0)        # per-layer cache block copy of the masked forward
        verify = L * (scratch + T * layer_row) + T * t_lm
        # draft: 1 row over the partial cache's draft view, all gamma+1 heads
        view = self.partial.draft_view(before_pos=ctx)
        m = len(view)
        req = S.ForwardRequest(tokens=[1], positions=[m], cache=view)
        t_d, _ = _t(lambda: self.model.forward(req))
        draft = t_d + (L - 1) * max(t_d - t_h, 0.0)
        # per-step cache maintenance: admit + draft view + reconcile, per layer
        part = self.partial
        pos_new = list(range(ctx - 4, ctx))
        t_adm, _ = _t(lambda: part.admit(pos_new, self.full))
        for layer in range(part.num_layers):  # undo (keeps the next sample's shapes)
            s = part.sink_size
            part.k[layer] = np.concatenate([part.k[layer][:s], part.k[layer][s + 4:]])
            part.v[layer] = np.concatenate([part.v[layer][:s], part.v[layer][s + 4:]])
            del part.positions[layer][s:s + 4]
            del part.scores[layer][s:s + 4]
        t_view, _ = _t(lambda: part.draft_view(before_pos=ctx))
        self.full.reserve(T)
        t_rec, _ = _t(lambda: self.full.reconcile(ctx - 4, [0, 1, 2, 3]))
        cache = L * (t_adm + t_view + t_rec)
        # verify sampling over T x V with the branch-extended windows
        logits = self.g.standard_normal((T, V)) * 3.0
        ns = types.SimpleNamespace(config=types.SimpleNamespace(sampler=self.smp),
                                   model=types.SimpleNamespace(config=types.SimpleNamespace(vocab_size=V)),
                                   window=self.window, depth=4)

        def sample_rows():
            masks = S.Session._node_masks(ns, self.tree)
            n = min(T, masks.shape[0])
            d = penalized_probs_masked(logits[:n], masks[:n], self.smp)
            for r in range(n):
                S.sample_at(S.truncate(d[r], self.smp.truncation), ctx + r, 0)
        t_s, _ = _t(sample_rows)
        hl = self.g.standard_normal((4, V))

        def topw():
            p = penalized_probs_masked(hl, np.broadcast_to(self.window.member_mask(), hl.shape), self.smp)
            return [np.argsort(-p[k], kind="stable")[:w] for k, w in enumerate((1, 3, 3, 3))]
        t_w, _ = _t(topw)

        def misc():
            self.ngrams.update([7, 8, 9, 10], [4, 5, 6])
            br = self.ngrams.retrieve(self.per_head[0][0], 20)
            br = [b for b in br if b[0] == self.per_head[0][0]]
            S.build_tree(self.per_head, br, S.TreeConfig((1, 3, 3, 3)))
        t_m, _ = _t(misc)
        ts, tp = self.refresh
        refresh = L * (ts + tp) * accepted / (c["B"] - c["S"] + 1)
        per_it = verify + draft + cache + t_s + t_w + t_m + refresh
        parts = {"verify_s": verify, "verify_scratch_per_layer_s": scratch, "verify_layer_row_s": layer_row,
                 "lm_head_row_s": t_lm, "draft_s": draft, "cache_maint_s": cache, "sample_s": t_s,
                 "draft_topw_s": t_w, "ngram_tree_s": t_m, "refresh_amortised_s": refresh,
                 "score_1layer_s": ts, "select_gather_1layer_s": tp, "draft_slots": m}
        return per_it, parts


def run(args, c, ctx, metric, workload, rows=41, accepted=4.0):
    """Print the reference arm's JSON line (rank 0 only)."""
    import json
    mod, where = import_reference()
    if mod is None:
        return None
    os.environ.setdefault("OMP_NUM_THREADS", str(host_cores()))
    cores = host_cores()
    line = {"metric": metric, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload, "ctx": ctx}}
    if args.config == "cfg1":
        steps = args.steps
        v, det = run_session(c, steps, args.warmup)
        sample = (f"reference swiftdec Session.step() end to end ({where}): prefill {c['prefix']}, "
                  f"{args.warmup} warm-up + {steps} timed iterations")
        line.update({"value": v, "steps": steps, "warmup": args.warmup, "ms_per_step": det["wall_s"] * 1e3 / steps,
                     "composed": False, "details": det})
    else:
        t0 = time.perf_counter()
        comp = Composer(c, ctx, rows=rows)
        warm = min(args.warmup, 1)  # one warm sample; each is ~5 s of CPU work at cfg3
        for _ in range(warm):
            comp.sample(accepted)
        per, parts_all, walls = [], [], []
        for _ in range(args.steps):
            w0 = time.perf_counter()
            s, parts = comp.sample(accepted)
            walls.append(time.perf_counter() - w0)
            per.append(s)
            parts_all.append(parts)
        per_it = statistics.median(per)
        v = accepted / per_it
        parts = {k: statistics.median(p[k] for p in parts_all) for k in parts_all[0]}
        sample = (f"reference swiftdec functions ({where}) at full {args.config} shapes, composed per iteration: "
                  f"{c['L']} x (verify layer: masked forward rows over ctx {ctx}, {rows} rows) + draft forward over "
                  f"{parts['draft_slots']} partial slots + cache maintenance + T x V sampling + top-w + n-gram/tree "
                  f"+ amortised refresh; {accepted:.2f} tokens/iteration; {args.steps} samples, median")
        line.update({"value": v, "steps": args.steps, "warmup": warm, "ms_per_step": per_it * 1e3,
                     "composed": True, "sample_wall_s": statistics.median(walls),
                     "setup_s": comp.setup_s, "run_wall_s": time.perf_counter() - t0,
                     "parts_s": {k: round(x, 5) for k, x in parts.items()}})
    line["cpu_baseline"] = {"value": line["value"], "unit": "tokens/s", "cores": cores, "kind": "reference",
                            "sample": sample}
    line["e2e"] = {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)
    return line
