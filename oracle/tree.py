"""Candidate tree (oracle; follows swiftdec/tree.py:76-175).

Head candidates form a Cartesian-product trie in DFS order; n-gram branches
join as chains merged greedily by token equality, exact duplicates dropped
while later branches keep their retrieval rank.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import product

import numpy as np


class WidthMismatch(ValueError):
    pass


class NGramLengthMismatch(ValueError):
    pass


@dataclass
class Path:
    tokens: tuple
    nodes: tuple
    origin: str
    origin_index: int


@dataclass
class Tree:
    tokens: list = field(default_factory=list)
    parent: list = field(default_factory=list)
    depth: list = field(default_factory=list)
    paths: list = field(default_factory=list)
    head_node_count: int = 0

    def __len__(self):
        return len(self.tokens)

    @property
    def mask(self) -> np.ndarray:
        return closure(self.parent)


def closure(parent) -> np.ndarray:
    """Reflexive ancestor closure: m[i, j] iff j is i or an ancestor (tree.py:76-84)."""
    n = len(parent)
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        j = i
        while j >= 0:
            m[i, j] = True
            j = parent[j]
    return m


def build_tree(per_head, grams=None, widths=None) -> Tree:
    """tree.py:87-175."""
    K = len(per_head)
    if widths is not None:
        if len(widths) != K:
            raise WidthMismatch("candidate lists vs widths")
        for k, c in enumerate(per_head):
            if len(c) != widths[k]:
                raise WidthMismatch("head width")
    t = Tree()
    kids: list[dict] = []
    roots: dict = {}

    def walk(seq):
        cur, nodes = -1, []
        for d, tok in enumerate(seq):
            table = roots if cur < 0 else kids[cur]
            nxt = table.get(tok)
            if nxt is None:
                nxt = len(t.tokens)
                t.tokens.append(tok)
                t.parent.append(cur)
                t.depth.append(d)
                kids.append({})
                table[tok] = nxt
            nodes.append(nxt)
            cur = nxt
        return tuple(nodes)

    seen = set()
    # itertools.product enumerates the Cartesian product in the same
    # lexicographic (DFS) order as the reference's recursive generator
    for rank, combo in enumerate(product(*per_head)):
        combo = tuple(int(x) for x in combo)
        t.paths.append(Path(combo, walk(combo), "head", rank))
        seen.add(combo)
    t.head_node_count = len(t.tokens)
    for rank, g in enumerate(grams or []):
        g = tuple(int(x) for x in g)
        if len(g) != K:
            raise NGramLengthMismatch("gram length")
        if per_head[0] and g[0] != per_head[0][0]:
            raise NGramLengthMismatch("gram anchor")
        if g in seen:
            continue
        seen.add(g)
        t.paths.append(Path(g, walk(g), "ngram", rank))
    return t
