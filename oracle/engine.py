"""Speculative session and AR oracle (oracle; follows swiftdec/engine.py).

Session.step is Algorithm 1 (engine.py:185-302): refresh check, draft forward
over the partial cache + penalised per-head top-w, n-gram retrieval, tree,
masked verification over the full cache, position-keyed sampling, exact-match
acceptance with a uniform pick among the longest paths, then reconcile /
admit / evict / window / n-gram commit.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import kvcache as kv
from .ngram import NGramTable
from .rng import derive_seed, uniform_at
from .sampling import (PenaltyWindow, SamplerConfig, node_masks, penalized_probs_masked,
                       sample_at, truncate)
from .tree import build_tree


class ConfigError(ValueError):
    pass


class PromptTooShort(ConfigError):
    pass


class SessionExhausted(RuntimeError):
    pass


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:59-85."""
    target_length: int
    sink_size: int = 32
    budget: int = 1024
    widths: tuple = (1, 3, 3, 3)
    k: int = 20
    sampler: SamplerConfig = field(default_factory=SamplerConfig)
    seed: int = 0
    bonus: bool = True

    def validate(self, gamma):
        if self.target_length < 1:
            raise ConfigError("target_length must be >= 1")
        if self.budget <= self.sink_size:
            raise ConfigError("budget must exceed sink_size")
        if self.budget - self.sink_size < gamma + 2:
            raise ConfigError("budget - sink_size must be at least gamma + 2")
        if len(self.widths) != gamma + 1:
            raise ConfigError("tree depth must equal gamma + 1")
        if self.k < 0:
            raise ConfigError("k must be >= 0")


@dataclass
class Record:
    """IterationRecord fields (metrics.py:29-44)."""
    step: int
    accepted: int
    ngram_accepted: int
    origin: str
    matched: int
    tokens: list
    refreshed: bool
    draft_ctx: int
    verify_ctx: int
    verify_rows: int
    path_index: int


def accept_paths(tree, y, select_seed, n, depth, bonus):
    """Exact-match validity, uniform pick among the longest (engine.py:247-274).
    Returns (pick, best_v, accepted, ys, keep)."""
    best_v, best = -1, []
    for idx, path in enumerate(tree.paths):
        expect, v = int(y[0]), 0
        for j, node in enumerate(path.nodes):
            if path.tokens[j] != expect:
                break
            v += 1
            expect = int(y[1 + node])
        if v > best_v:
            best_v, best = v, [idx]
        elif v == best_v:
            best.append(idx)
    pick = best[int(uniform_at(select_seed, n) * len(best))]
    chosen = tree.paths[pick]
    accepted = min(best_v + 1, depth) if bonus else max(best_v, 1)
    ys = ([int(y[0])] + [int(y[1 + nd]) for nd in chosen.nodes[: accepted - 1]])[:accepted]
    keep = [0] + [1 + nd for nd in chosen.nodes[: accepted - 1]]
    return pick, best_v, accepted, ys, keep


class Session:
    def __init__(self, model, prompt, config: EngineConfig):
        gamma = model.config.gamma
        config.validate(gamma)
        if len(prompt) <= config.sink_size:
            raise PromptTooShort("prompt must exceed the sink size")
        self.model, self.config = model, config
        self.gamma, self.depth = gamma, gamma + 1
        self.tokens = [int(t) for t in prompt]
        self.emitted: list[int] = []
        self.records: list[Record] = []
        self.window = PenaltyWindow(config.sampler.window, model.config.vocab_size)
        self.ngrams = NGramTable(n=self.depth, k_max=max(64, config.k))
        self.select_seed = derive_seed(config.seed, "branch-select")
        self.full = model.new_cache()
        _, q = model.forward(self.tokens, list(range(len(prompt))), self.full, heads_needed=1)
        self.last_queries = q.sum(axis=0)
        self.partial = self._build_partial(len(prompt) - 1)

    def body_scores(self, upto):
        c, s = self.model.config, self.config.sink_size
        return np.stack([
            kv.importance_scores(self.last_queries[l], self.full.k_raw[l, s:upto], c.group_size)
            for l in range(c.num_layers)
        ])

    def _build_partial(self, upto):
        cfg = self.config
        if upto < cfg.budget:
            return kv.mirror_partial(self.full, cfg.sink_size, cfg.budget, upto=upto)
        return kv.prefill_partial(self.full, cfg.sink_size, cfg.budget, self.body_scores(upto), upto=upto)

    @property
    def done(self):
        return len(self.emitted) >= self.config.target_length

    def draft(self, n):
        """Draft forward + penalised per-head top-w (engine.py:199-217)."""
        cfg = self.config
        ks, vs = self.partial.draft_view(n - 1)
        buf = self.model.buffer_from_view(ks, vs)
        m = len(buf)
        bundles, _ = self.model.forward([self.tokens[-1]], [m], buf)
        head_logits = bundles[0]
        member = np.broadcast_to(self.window.member_mask(), head_logits.shape)
        probs = penalized_probs_masked(head_logits, member, cfg.sampler)
        per_head = [[int(t) for t in np.argsort(-probs[k], kind="stable")[: cfg.widths[k]]]
                    for k in range(self.depth)]
        return m, head_logits, per_head

    def step(self):
        if self.done:
            raise SessionExhausted("target reached")
        cfg, smp = self.config, self.config.sampler
        n = len(self.tokens)
        pending = self.tokens[-1]
        refreshed = kv.needs_refresh(len(self.full), self.partial)
        if refreshed:
            self.partial = self._build_partial(len(self.full))
        m, _, per_head = self.draft(n)
        grams = self.ngrams.retrieve(per_head[0][0], cfg.k)
        tree = build_tree(per_head, grams, cfg.widths)
        base = n - 1
        if len(self.full) > base:
            self.full.truncate(base)
        rows = 1 + len(tree)
        mask = np.zeros((rows, base + rows), dtype=bool)
        mask[:, : base + 1] = True
        mask[1:, base + 1:] = tree.mask
        positions = [n - 1] + [n + d for d in tree.depth]
        bundles, q = self.model.forward([pending] + tree.tokens, positions, self.full, mask, heads_needed=1)
        dists = penalized_probs_masked(bundles[:, 0, :], node_masks(self.window, tree.tokens, tree.parent, self.depth), smp)
        y = np.empty(rows, dtype=np.int64)
        for r in range(rows):
            pos = n if r == 0 else n + tree.depth[r - 1] + 1
            y[r] = sample_at(truncate(dists[r], smp.truncation), pos, smp.seed)
        pick, best_v, accepted, ys, keep = accept_paths(tree, y, self.select_seed, n, self.depth, cfg.bonus)
        self.full.reconcile(base, keep)
        self.last_queries = q[keep].sum(axis=0)
        self.partial.admit(list(range(n - 1, n - 1 + accepted)), self.full)
        kv.evict_to_budget(self.partial, protected=accepted)
        tail = self.emitted[max(0, len(self.emitted) - (self.depth - 1)):]
        self.tokens += ys
        self.emitted += ys
        for t in ys:
            self.window.push(t)
        self.ngrams.update(ys, tail)
        origin = tree.paths[pick].origin
        rec = Record(len(self.records), accepted,
                     accepted if (origin == "ngram" and best_v == self.depth) else 0,
                     origin, best_v, ys, refreshed, m, base, rows, pick)
        self.records.append(rec)
        self.last_tree, self.last_y = tree, y
        return rec


def generate(model, prompt, config):
    s = Session(model, prompt, config)
    while not s.done:
        s.step()
    return s.emitted, s


def generate_ar(model, prompt, config: EngineConfig):
    """Plain decoding with the same sampler and position keys (engine.py:328-360)."""
    config.validate(model.config.gamma)
    if len(prompt) <= config.sink_size:
        raise PromptTooShort("prompt must exceed the sink size")
    smp = config.sampler
    cache = model.new_cache()
    b, _ = model.forward(list(prompt), list(range(len(prompt))), cache, heads_needed=1)
    logits = b[-1, 0]
    window = PenaltyWindow(smp.window, model.config.vocab_size)
    toks, out = list(prompt), []
    while True:
        d = penalized_probs_masked(logits, window.member_mask(), smp)
        t = sample_at(truncate(d, smp.truncation), len(toks), smp.seed)
        out.append(t)
        window.push(t)
        toks.append(t)
        if len(out) >= config.target_length:
            return out
        b, _ = model.forward([t], [len(toks) - 1], cache, heads_needed=1)
        logits = b[-1, 0]
