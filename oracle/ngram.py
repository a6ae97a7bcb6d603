"""Exact n-gram counts over generated tokens (oracle; follows swiftdec/ngram.py:18-66).

Every window of length n ending inside the newly committed span is counted;
each counted window stamps a global clock. Retrieval ranks the grams sharing a
first token by (frequency desc, last-stamp desc).
"""

from __future__ import annotations


class NGramTable:
    def __init__(self, n: int = 4, k_max: int = 64):
        if n < 1:
            raise ValueError("n must be >= 1")
        self.n = n
        self.k_max = k_max
        self.freq: dict[tuple, int] = {}
        self.last: dict[tuple, int] = {}
        self.by_first: dict[int, set] = {}
        self.clock = 0

    def __len__(self):
        return len(self.freq)

    def frequency(self, gram) -> int:
        return self.freq.get(tuple(gram), 0)

    def update(self, new, tail) -> None:
        seq = [int(x) for x in tail] + [int(x) for x in new]
        for end in range(len(tail), len(seq)):
            start = end + 1 - self.n
            if start < 0:
                continue
            g = tuple(seq[start:end + 1])
            self.clock += 1
            self.freq[g] = self.freq.get(g, 0) + 1
            self.last[g] = self.clock
            self.by_first.setdefault(g[0], set()).add(g)

    def retrieve(self, first: int, k: int) -> list[tuple]:
        if k > self.k_max:
            raise ValueError("k exceeds k_max")
        if k <= 0:
            return []
        cands = self.by_first.get(int(first), ())
        return sorted(cands, key=lambda g: (-self.freq[g], -self.last[g]))[:k]
