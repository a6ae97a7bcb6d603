"""Full / partial KV caches (oracle; follows swiftdec/kvcache.py).

FullCache: append-only per-layer K_raw, K_rot, V with staging beyond the
committed length (kvcache.py:71-133). PartialCache: sink + importance-ordered
body (kvcache.py:191-240). Eq. 2 scoring (kvcache.py:243-265), top-K build
(kvcache.py:268-297), mirror build (kvcache.py:300-319), refresh trigger
(kvcache.py:322-324), eviction (kvcache.py:332-354).
"""

from __future__ import annotations

import numpy as np


class GroupMismatch(ValueError):
    pass


class BudgetTooSmall(ValueError):
    pass


class SinkViolation(RuntimeError):
    pass


class FullCache:
    def __init__(self, num_layers, num_kv_heads, head_dim, cap=64):
        self.num_layers, self.num_kv_heads, self.head_dim = num_layers, num_kv_heads, head_dim
        self.positions: list[int] = []
        shape = (num_layers, cap, num_kv_heads, head_dim)
        self.k_raw = np.zeros(shape)
        self.k_rot = np.zeros(shape)
        self.v = np.zeros(shape)

    def __len__(self):
        return len(self.positions)

    def reserve(self, extra):
        need = len(self) + extra
        cap = self.k_raw.shape[1]
        if need <= cap:
            return
        while cap < need:
            cap *= 2
        for name in ("k_raw", "k_rot", "v"):
            old = getattr(self, name)
            new = np.zeros((old.shape[0], cap) + old.shape[2:])
            new[:, : len(self)] = old[:, : len(self)]
            setattr(self, name, new)

    def stage_rows(self, layer, k_raw, k_rot, v):
        """Write T staged rows after the committed length (kvcache.py:91-96)."""
        n = len(self)
        t = k_raw.shape[0]
        self.k_raw[layer, n:n + t] = k_raw
        self.k_rot[layer, n:n + t] = k_rot
        self.v[layer, n:n + t] = v

    def commit_rows(self, positions):
        self.positions.extend(int(p) for p in positions)

    def truncate(self, n):
        del self.positions[n:]

    def reconcile(self, base_len, keep_offsets):
        """kvcache.py:116-127 (fancy-index copy: reads before writes)."""
        keep = [base_len + o for o in keep_offsets]
        end = base_len + len(keep)
        for arr in (self.k_raw, self.k_rot, self.v):
            arr[:, base_len:end] = arr[:, keep]
        self.positions = self.positions[:base_len] + [self.positions[i] for i in keep]

    def gather(self, layer, positions):
        idx = np.asarray(positions, dtype=np.intp)
        return self.k_raw[layer, idx].copy(), self.v[layer, idx].copy()


def importance_scores(queries, keys, group_size):
    """Eq. 2: score_n = sum_k sum_g q[k*G+g] . K[n, k] (kvcache.py:243-265)."""
    q = np.asarray(queries, dtype=np.float64)
    k = np.asarray(keys, dtype=np.float64)
    single = k.ndim == 2
    if single:
        k = k[None]
    H, dh = q.shape
    if H != group_size * k.shape[1]:
        raise GroupMismatch("query heads vs kv heads * group")
    qg = q.reshape(k.shape[1], group_size, dh).sum(axis=1)  # (Hk, dh)
    s = np.einsum("kd,nkd->n", qg, k)
    return s[0] if single else s


class PartialCache:
    def __init__(self, sink_size, budget, positions, k, v, scores, mark):
        if budget <= sink_size:
            raise BudgetTooSmall("budget must exceed sink")
        self.sink_size, self.budget = sink_size, budget
        self.positions, self.k, self.v, self.scores, self.mark = positions, k, v, scores, mark

    @property
    def num_layers(self):
        return len(self.positions)

    def __len__(self):
        return len(self.positions[0]) if self.positions else 0

    @property
    def capacity(self):
        return self.budget - self.sink_size

    def admit(self, positions, full: FullCache):
        """New entries at the body head (kvcache.py:215-225)."""
        if not positions:
            return
        s = self.sink_size
        for l in range(self.num_layers):
            kn, vn = full.gather(l, positions)
            self.k[l] = np.concatenate([self.k[l][:s], kn, self.k[l][s:]])
            self.v[l] = np.concatenate([self.v[l][:s], vn, self.v[l][s:]])
            self.positions[l][s:s] = list(positions)
            self.scores[l][s:s] = [None] * len(positions)

    def draft_view(self, before_pos):
        """Entries with pos < before_pos sorted by position (kvcache.py:227-240).
        Returns per-layer (k_raw, v) arrays; rank = row index."""
        ks, vs = [], []
        for l in range(self.num_layers):
            idx = sorted((p, i) for i, p in enumerate(self.positions[l]) if p < before_pos)
            sel = np.asarray([i for _, i in idx], dtype=np.intp)
            ks.append(self.k[l][sel])
            vs.append(self.v[l][sel])
        return ks, vs


def select_body(scores_row, sink_size, n, take):
    """Top-`take` of positions [sink, n) by (-score, pos) (kvcache.py:286-287)."""
    sc = np.asarray(scores_row, dtype=np.float64)
    pos = np.arange(sink_size, n)
    order = np.lexsort((pos, -sc))  # primary -score, secondary pos
    return [int(pos[i]) for i in order[:take]]


def prefill_partial(full: FullCache, sink_size, budget, scores, upto=None):
    """kvcache.py:268-297."""
    n = len(full) if upto is None else upto
    if budget <= sink_size:
        raise BudgetTooSmall("budget must exceed sink")
    if n < budget:
        raise ValueError("prefill_partial needs at least budget entries")
    scores = np.asarray(scores, dtype=np.float64)
    take = budget - sink_size
    P, K, V, S = [], [], [], []
    for l in range(full.num_layers):
        body = select_body(scores[l], sink_size, n, take)
        pos = list(range(sink_size)) + body
        k, v = full.gather(l, pos)
        P.append(pos)
        K.append(k)
        V.append(v)
        S.append([None] * sink_size + [float(scores[l][p - sink_size]) for p in body])
    return PartialCache(sink_size, budget, P, K, V, S, mark=n)


def mirror_partial(full: FullCache, sink_size, budget, upto=None):
    """Newest-first mirror for short prefixes (kvcache.py:300-319)."""
    n = len(full) if upto is None else upto
    if budget <= sink_size:
        raise BudgetTooSmall("budget must exceed sink")
    P, K, V, S = [], [], [], []
    for l in range(full.num_layers):
        pos = list(range(sink_size)) + list(range(n - 1, sink_size - 1, -1))
        k, v = full.gather(l, pos)
        P.append(pos)
        K.append(k)
        V.append(v)
        S.append([None] * len(pos))
    return PartialCache(sink_size, budget, P, K, V, S, mark=n)


def needs_refresh(full_len, partial: PartialCache) -> bool:
    return (full_len - partial.mark) > partial.capacity


def evict_to_budget(partial: PartialCache, protected=0):
    """Trim the body tail back to the budget (kvcache.py:332-354)."""
    over = len(partial) - partial.budget
    if over <= 0:
        return partial
    if len(partial) - partial.sink_size - over < protected:
        raise SinkViolation("eviction would reach protected entries")
    keep = len(partial) - over
    for l in range(partial.num_layers):
        partial.k[l] = partial.k[l][:keep]
        partial.v[l] = partial.v[l][:keep]
        del partial.positions[l][keep:]
        del partial.scores[l][keep:]
    return partial
