"""Run metrics (mirrors swiftdec/metrics.py:29-140; reporting only, host side).

alpha (Eq. 5) = sum(a_i) / ((gamma + 1) * iterations); beta (Eq. 7) credits an
iteration whose chosen path was an n-gram branch accepted in full.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import Iterable


class SequenceTooShort(ValueError):
    pass


@dataclass
class IterationRecord:
    step: int
    accepted: int
    ngram_accepted: int
    origin: str
    matched: int
    tokens: list[int]
    forwards: int = 2
    refreshed: bool = False
    draft_ctx: int = 0
    verify_ctx: int = 0
    verify_rows: int = 0
    path_index: int = 0

    def to_json(self) -> str:
        return json.dumps(asdict(self))

    @classmethod
    def from_json(cls, line: str) -> "IterationRecord":
        return cls(**json.loads(line))


@dataclass
class RunMetrics:
    iterations: int
    gamma: int
    accepted: list[int]
    ngram_accepted: list[int]
    alpha: float
    beta: float
    emitted: int
    distinct: dict[int, float]
    forward_counts: dict[str, int] = field(default_factory=dict)
    wall_times: dict[str, float] = field(default_factory=dict)

    def to_dict(self) -> dict:
        d = asdict(self)
        d["distinct"] = {str(k): v for k, v in self.distinct.items()}
        return d


def acceptance_rate(records: Iterable[IterationRecord], gamma: int) -> float:
    recs = list(records)
    if not recs:
        raise ValueError("acceptance rate needs at least one iteration")
    return sum(r.accepted for r in recs) / ((gamma + 1) * len(recs))


def ngram_acceptance_rate(records: Iterable[IterationRecord], gamma: int) -> float:
    recs = list(records)
    if not recs:
        raise ValueError("acceptance rate needs at least one iteration")
    return sum(r.ngram_accepted for r in recs) / ((gamma + 1) * len(recs))


def speedup(ar_cost: float, swift_cost: float) -> float:
    if ar_cost <= 0 or swift_cost <= 0:
        raise ValueError("latencies must be positive")
    return ar_cost / swift_cost


def distinct_n(tokens: list[int], n: int) -> float:
    if len(tokens) < n:
        raise SequenceTooShort(f"{len(tokens)} tokens cannot form an {n}-gram")
    windows = len(tokens) - n + 1
    return len({tuple(tokens[i:i + n]) for i in range(windows)}) / windows


def distinct_average(tokens, ns=(1, 2, 3, 4)) -> dict[int, float]:
    return {n: distinct_n(tokens, n) for n in ns if len(tokens) >= n}


def collect_metrics(records, gamma, emitted_tokens, forward_counts=None, wall_times=None) -> RunMetrics:
    return RunMetrics(
        iterations=len(records), gamma=gamma, accepted=[r.accepted for r in records],
        ngram_accepted=[r.ngram_accepted for r in records], alpha=acceptance_rate(records, gamma),
        beta=ngram_acceptance_rate(records, gamma), emitted=len(emitted_tokens),
        distinct=distinct_average(emitted_tokens), forward_counts=forward_counts or {},
        wall_times=wall_times or {},
    )


def write_trace(records, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for rec in records:
            fh.write(rec.to_json() + "\n")


def read_trace(path) -> list[IterationRecord]:
    return [IterationRecord.from_json(line) for line in Path(path).read_text(encoding="utf-8").splitlines()
            if line.strip()]
