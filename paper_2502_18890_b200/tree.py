"""Candidate tree (API mirror of swiftdec/tree.py, built on device).

`build_tree` validates on the host exactly like the reference
(tree.py:98-106, 155-161) and then runs the single-CTA builder
`sd_tree_build` (csrc/step.cu): Cartesian-product head trie in DFS order plus
greedily merged n-gram chains, with the ancestor-closure mask.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


class WidthMismatch(ValueError):
    """Per-head candidate lists disagree with the configured widths."""


class NGramLengthMismatch(ValueError):
    """An n-gram branch is not exactly tree-depth long."""


@dataclass(frozen=True)
class TreeConfig:
    widths: tuple[int, ...] = (1, 3, 3, 3)

    def __post_init__(self) -> None:
        if not self.widths or any(w < 1 for w in self.widths):
            raise ValueError("widths must be a non-empty list of counts >= 1")

    @property
    def depth(self) -> int:
        return len(self.widths)

    @property
    def head_leaves(self) -> int:
        return int(np.prod(self.widths))

    @property
    def head_nodes(self) -> int:
        total, run = 0, 1
        for w in self.widths:
            run *= w
            total += run
        return total

    def max_rows(self, k: int) -> int:
        """1 + head nodes + k n-gram chains of depth-1 fresh nodes each."""
        return 1 + self.head_nodes + k * max(0, self.depth - 1)

    @classmethod
    def parse(cls, text: str) -> "TreeConfig":
        return cls(tuple(int(w) for w in text.split(",")))


@dataclass
class PathInfo:
    tokens: tuple[int, ...]
    nodes: tuple[int, ...]
    origin: str
    origin_index: int


@dataclass
class CandidateTree:
    tokens: list[int]
    parent: list[int]
    depth: list[int]
    mask: np.ndarray
    paths: list[PathInfo]
    head_node_count: int = 0

    def __len__(self) -> int:
        return len(self.tokens)

    def position_offsets(self) -> list[int]:
        return list(self.depth)


def closure_mask(parent) -> np.ndarray:
    n = len(parent)
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        j = i
        while j != -1:
            m[i, j] = True
            j = parent[j]
    return m


def tree_from_record(rec) -> CandidateTree:
    """Materialise the device tree record (int32 words) as a CandidateTree."""
    lay = L.tree_layout()
    r = rec.cpu().numpy() if isinstance(rec, torch.Tensor) else np.asarray(rec)
    T = int(r[lay["T"]])
    nodes = T - 1
    K = int(r[lay["DEPTH"]])
    tokens = [int(x) for x in r[lay["TOK"] + 1: lay["TOK"] + 1 + nodes]]
    parent = [int(x) for x in r[lay["PARENT"]: lay["PARENT"] + nodes]]
    depth = [int(x) for x in r[lay["NDEPTH"]: lay["NDEPTH"] + nodes]]
    paths = []
    for p in range(int(r[lay["NPATHS"]])):
        nd = tuple(int(x) for x in r[lay["PNODES"] + p * L.TREE_MAX_DEPTH: lay["PNODES"] + p * L.TREE_MAX_DEPTH + K])
        origin = "ngram" if int(r[lay["PORIGIN"] + p]) else "head"
        paths.append(PathInfo(tuple(tokens[i] for i in nd), nd, origin, int(r[lay["POIDX"] + p])))
    mw = L.MASK_WORDS
    mask = np.zeros((nodes, nodes), dtype=bool)
    for i in range(nodes):
        words = r[lay["MASK"] + (i + 1) * mw: lay["MASK"] + (i + 2) * mw].astype(np.int64) & 0xFFFFFFFF
        for j in range(nodes):
            mask[i, j] = bool((int(words[(j + 1) >> 5]) >> ((j + 1) & 31)) & 1)
    return CandidateTree(tokens, parent, depth, mask, paths, int(r[lay["HEADNODES"]]))


def build_tree(per_head_topk, ngram_branches=None, widths: TreeConfig | None = None) -> CandidateTree:
    K = len(per_head_topk)
    if widths is not None:
        if widths.depth != K:
            raise WidthMismatch(f"{K} candidate lists for widths {widths.widths}")
        for k, c in enumerate(per_head_topk):
            if len(c) != widths.widths[k]:
                raise WidthMismatch(f"head {k} has {len(c)} candidates, widths want {widths.widths[k]}")
    grams = [tuple(int(t) for t in g) for g in (ngram_branches or [])]
    for g in grams:
        if len(g) != K:
            raise NGramLengthMismatch(f"branch {g} has length {len(g)}, tree depth is {K}")
        if per_head_topk[0] and g[0] != per_head_topk[0][0]:
            raise NGramLengthMismatch(f"branch {g} does not start at the head argmax {per_head_topk[0][0]}")
    if K > L.TREE_MAX_DEPTH:
        raise ValueError(f"tree depth {K} > {L.TREE_MAX_DEPTH}")
    ws = [len(c) for c in per_head_topk]
    cfg = TreeConfig(tuple(ws))
    if cfg.max_rows(len(grams)) > L.TREE_MAX_ROWS or cfg.head_leaves + len(grams) > L.TREE_MAX_PATHS:
        raise ValueError("tree exceeds device capacity")
    L.require_cuda()
    dev = torch.device("cuda")
    flat = torch.tensor([int(t) for c in per_head_topk for t in c], dtype=torch.int32, device=dev)
    g = torch.tensor(grams if grams else [[0] * K], dtype=torch.int32, device=dev).reshape(-1)
    rec = torch.zeros(L.tree_layout()["TOTAL"], dtype=torch.int32, device=dev)
    L.call("sd_tree_build", L.ptr(flat), L.host_i32(ws), K, L.ptr(g), None, len(grams), None, 0, L.ptr(rec),
           L.stream())
    return tree_from_record(rec)


def mask_check(tree: CandidateTree) -> bool:
    return bool(np.array_equal(tree.mask, closure_mask(tree.parent)))
