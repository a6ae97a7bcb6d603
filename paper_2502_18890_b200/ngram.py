"""Token reutilisation table on device (API mirror of swiftdec/ngram.py:18-66).

A hashed device table (open addressing over n-token keys, per-first-token
chains, exact counts and a global recency clock) updated in place by
`sd_ngram_update` / the step's commit kernel. Retrieval returns the top-k grams
starting with a token by (frequency desc, last-seen desc).
"""

from __future__ import annotations

import torch

from . import _lib as L


class NGramTable:
    def __init__(self, n: int = 4, k_max: int = 64, capacity: int = 1 << 16, vocab_size: int = 1 << 18,
                 device: str | torch.device = "cuda"):
        if n < 1:
            raise ValueError("n must be >= 1")
        if k_max > 64:
            raise ValueError("k_max above the device limit of 64")
        L.require_cuda()
        cap = 1
        while cap < max(2, capacity):
            cap <<= 1
        self.n, self.k_max, self.capacity, self.vocab_size = n, k_max, cap, vocab_size
        self.device = torch.device(device)
        nbytes = L.load().sd_ngram_bytes(n, cap, vocab_size)
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        L.call("sd_ngram_init", L.ptr(self.buf), n, cap, vocab_size, L.stream())

    @property
    def handle(self) -> int:
        return self.buf.data_ptr()

    def __len__(self) -> int:
        out = torch.empty(1, dtype=torch.int32, device=self.device)
        L.call("sd_ngram_size", self.handle, L.ptr(out), L.stream())
        return int(out.item())

    def overflowed(self) -> bool:
        return bool(self.buf[:64].view(torch.int64)[5].item())

    def frequency(self, gram) -> int:
        g = torch.tensor([int(x) for x in gram], dtype=torch.int32, device=self.device)
        if g.numel() != self.n:
            return 0
        out = torch.empty(1, dtype=torch.int32, device=self.device)
        L.call("sd_ngram_frequency", self.handle, L.ptr(g), 1, L.ptr(out), L.stream())
        return int(out.item())

    def _check(self, toks):
        for t in toks:
            if not 0 <= int(t) < self.vocab_size:
                raise ValueError(f"token {t} outside the table vocabulary {self.vocab_size}")

    def update(self, newly_committed, history_tail) -> None:
        seq = [int(t) for t in history_tail] + [int(t) for t in newly_committed]
        if not seq:
            return
        self._check(seq)
        s = torch.tensor(seq, dtype=torch.int32, device=self.device)
        L.call("sd_ngram_update", self.handle, L.ptr(s), len(history_tail), len(newly_committed), L.stream())

    def retrieve(self, first_token: int, k: int) -> list[tuple[int, ...]]:
        if k > self.k_max:
            raise ValueError(f"k {k} exceeds k_max {self.k_max}")
        if k <= 0:
            return []
        if not 0 <= int(first_token) < self.vocab_size:
            return []
        f = torch.tensor([int(first_token)], dtype=torch.int32, device=self.device)
        out = torch.empty((k, self.n), dtype=torch.int32, device=self.device)
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        L.call("sd_ngram_retrieve", self.handle, L.ptr(f), k, L.ptr(out), L.ptr(cnt), L.stream())
        c = int(cnt.item())
        return [tuple(int(x) for x in row) for row in out[:c].cpu().tolist()]
