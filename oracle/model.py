"""TinyTransformer forward in float64 (oracle; follows swiftdec/model.py:150-313).

Pre-norm rotary GQA transformer, tied embedding / LM head, non-gated SiLU MLP
of width 4d, gamma residually chained draft heads (model.py:104-120).
The restatement is vectorised over rows; the reference loops row by row.
Visibility per row is identical: cache + masked ancestors + self
(model.py:290-300) or cache + causal prefix (model.py:301-305).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kvcache import FullCache


class PositionOverflow(ValueError):
    pass


class MaskShapeMismatch(ValueError):
    pass


@dataclass(frozen=True)
class ModelConfig:
    """model.py:44-75."""
    vocab_size: int
    num_layers: int = 2
    hidden_dim: int = 64
    num_heads: int = 4
    num_kv_heads: int = 4
    gamma: int = 3
    max_positions: int = 65536
    init_seed: int = 0

    @property
    def head_dim(self):
        return self.hidden_dim // self.num_heads

    @property
    def group_size(self):
        return self.num_heads // self.num_kv_heads


def param_specs(c: ModelConfig):
    """Names, shapes and init scales in reference order (model.py:173-193)."""
    d, H, Hk, dh = c.hidden_dim, c.num_heads, c.num_kv_heads, c.head_dim
    specs = [("embed", (c.vocab_size, d), 0.3)]
    for i in range(c.num_layers):
        specs += [
            (f"l{i}.ln1", (d,), 0.0), (f"l{i}.wq", (d, H * dh), d ** -0.5),
            (f"l{i}.wk", (d, Hk * dh), d ** -0.5), (f"l{i}.wv", (d, Hk * dh), d ** -0.5),
            (f"l{i}.wo", (H * dh, d), (H * dh) ** -0.5), (f"l{i}.ln2", (d,), 0.0),
            (f"l{i}.w1", (d, 4 * d), d ** -0.5), (f"l{i}.w2", (4 * d, d), (4 * d) ** -0.5),
        ]
    specs.append(("ln_f", (d,), 0.0))
    specs += [(f"head{i + 1}", (d, d), 0.3 * d ** -0.5) for i in range(c.gamma)]
    return specs


def init_params(c: ModelConfig):
    """Seeded per-tensor streams: SeedSequence(init_seed, spawn_key=(idx,)) (model.py:195-205)."""
    out = {}
    for idx, (name, shape, scale) in enumerate(param_specs(c)):
        if scale == 0.0:
            out[name] = np.ones(shape)
        else:
            g = np.random.default_rng(np.random.SeedSequence(entropy=c.init_seed, spawn_key=(idx,)))
            out[name] = g.normal(0.0, scale, size=shape)
    return out


def rope(rows, positions, inv_freq):
    """Interleaved-pair rotation, fp64 angles (model.py:216-232)."""
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = rows[..., 0::2], rows[..., 1::2]
    out = np.empty_like(rows)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


def rmsnorm(x, gain):
    """model.py:234-236, row-wise."""
    ms = np.einsum("...d,...d->...", x, x)[..., None] / x.shape[-1]
    return x * (gain / np.sqrt(ms + 1e-6))


class TinyTransformer:
    def __init__(self, config: ModelConfig, params=None):
        self.config = c = config
        self.inv_freq = 10000.0 ** (-np.arange(0, c.head_dim, 2) / c.head_dim)
        self.params = params if params is not None else init_params(c)
        self.scale = 1.0 / np.sqrt(c.head_dim)

    def new_cache(self):
        c = self.config
        return FullCache(c.num_layers, c.num_kv_heads, c.head_dim)

    def buffer_from_view(self, ks, vs):
        """Draft view as a cache whose keys are rotated at rank 0..m-1
        (kvcache.py:136-165)."""
        c = self.config
        m = ks[0].shape[0]
        buf = FullCache(c.num_layers, c.num_kv_heads, c.head_dim, cap=max(m + 8, 8))
        ranks = np.arange(m)
        for l in range(c.num_layers):
            buf.k_raw[l, :m] = ks[l]
            buf.k_rot[l, :m] = rope(ks[l], ranks, self.inv_freq) if m else ks[l]
            buf.v[l, :m] = vs[l]
        buf.positions = list(range(m))
        return buf

    def chained_logits(self, h0, heads):
        """Eq. 1 residual chain, l_i = E h_i (model.py:104-120)."""
        p = self.params
        hs = [h0]
        for i in range(heads - 1):
            hs.append(hs[-1] @ p[f"head{i + 1}"] + hs[-1])
        return np.stack([h @ p["embed"].T for h in hs], axis=-2)

    def forward(self, tokens, positions, cache, mask=None, heads_needed=None, logit_rows=None):
        """Returns (bundles (T, gamma+1, V), queries (T, L, H, dh) pre-rotation).
        logit_rows (test convenience, not in the reference): compute the head
        logits only for these rows (the others stay -inf), so a teacher-forced
        check over a long sequence does not materialise T x V logits it ignores."""
        c, p = self.config, self.params
        T = len(tokens)
        if T == 0:
            raise ValueError("empty request")
        if len(positions) != T:
            raise ValueError("tokens/positions length")
        if max(positions) >= c.max_positions:
            raise PositionOverflow("position >= max_positions")
        ctx = len(cache)
        if mask is not None:
            mask = np.asarray(mask, dtype=bool)
            if mask.shape != (T, ctx + T):
                raise MaskShapeMismatch(f"mask {mask.shape} vs {(T, ctx + T)}")
        cache.reserve(T)
        Hk, G, dh, H = c.num_kv_heads, c.group_size, c.head_dim, c.num_heads
        # visibility over [cache, request rows]
        vis = np.zeros((T, ctx + T), dtype=bool)
        vis[:, :ctx] = True
        tri = np.tril(np.ones((T, T), dtype=bool))
        vis[:, ctx:] = (mask[:, ctx:] & tri) if mask is not None else tri
        vis[np.arange(T), ctx + np.arange(T)] = True
        h = p["embed"][np.asarray(tokens)].astype(np.float64)
        queries = np.empty((T, c.num_layers, H, dh))
        pos = np.asarray(positions)
        for l in range(c.num_layers):
            x = rmsnorm(h, p[f"l{l}.ln1"])
            q = (x @ p[f"l{l}.wq"]).reshape(T, H, dh)
            k = (x @ p[f"l{l}.wk"]).reshape(T, Hk, dh)
            v = (x @ p[f"l{l}.wv"]).reshape(T, Hk, dh)
            queries[:, l] = q
            k_rot = rope(k, pos, self.inv_freq)
            q_rot = rope(q, pos, self.inv_freq) * self.scale
            cache.stage_rows(l, k, k_rot, v)
            K = cache.k_rot[l, : ctx + T]
            V = cache.v[l, : ctx + T]
            s = np.einsum("tkgd,nkd->tkgn", q_rot.reshape(T, Hk, G, dh), K)
            s = np.where(vis[:, None, None, :], s, -np.inf)
            s = np.exp(s - s.max(axis=-1, keepdims=True))
            w = s / s.sum(axis=-1, keepdims=True)
            o = np.einsum("tkgn,nkd->tkgd", w, V).reshape(T, H * dh)
            h = h + o @ p[f"l{l}.wo"]
            a = rmsnorm(h, p[f"l{l}.ln2"]) @ p[f"l{l}.w1"]
            h = h + (a / (1.0 + np.exp(-a))) @ p[f"l{l}.w2"]
        h0 = rmsnorm(h, p["ln_f"])
        heads = c.gamma + 1 if heads_needed is None else min(heads_needed, c.gamma + 1)
        if logit_rows is None:
            bundles = np.full((T, c.gamma + 1, c.vocab_size), -np.inf)
            bundles[:, :heads] = self.chained_logits(h0, heads)
        else:
            rows = np.asarray(logit_rows, dtype=np.int64)
            bundles = np.full((len(rows), c.gamma + 1, c.vocab_size), -np.inf)
            bundles[:, :heads] = self.chained_logits(h0[rows], heads)
        cache.commit_rows(positions)
        return bundles, queries
