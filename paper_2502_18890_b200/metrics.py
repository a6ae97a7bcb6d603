"""Per-iteration records, run statistics, trace files and a B200 cost model.

Same public names and meaning as swiftdec/metrics.py (IterationRecord
fields 29-44, RunMetrics 47-62, the acceptance rates of Eq. 5 / Eq. 7,
distinct-n, JSONL traces, CostParams and the simulated speedup 143-213), so
the reference's `report` / `bench` tooling reads device runs unchanged.
The implementation is array based: a run's records become one int64 matrix
(`record_matrix`) from which alpha, beta and the cost-model replay are
computed with numpy, and distinct-n counts unique rows of a sliding-window
view instead of building Python tuples.

`B200` is a CostParams preset for one B200 running the bench's cfg3 model
(MEASURED_PEAKS.json-style HBM figure, dense bf16 peak, 12.43 GB of
reference-architecture weights, 131072 B of K/V per token) and
`forward_bytes` / `step_bound_seconds` give the per-iteration HBM bound the
bench's roofline discussion uses.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field, fields
from pathlib import Path
from typing import Iterable

import numpy as np


class SequenceTooShort(ValueError):
    """Fewer tokens than the n-gram size."""


_RECORD_FIELDS = ("step", "accepted", "ngram_accepted", "origin", "matched", "tokens", "forwards", "refreshed",
                  "draft_ctx", "verify_ctx", "verify_rows", "path_index")


@dataclass
class IterationRecord:
    """One decode iteration (engine.py:293-302): a_i (bonus included), b_i
    (full credit or 0), the winning branch's origin and draft matches, the
    committed tokens, and the cache sizes / rows the two forwards touched."""

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
        return json.dumps({k: getattr(self, k) for k in _RECORD_FIELDS})

    @classmethod
    def from_json(cls, line: str) -> "IterationRecord":
        raw = json.loads(line)
        known = {f.name for f in fields(cls)}
        return cls(**{k: v for k, v in raw.items() if k in known})


# columns of record_matrix
COL_ACCEPTED, COL_NGRAM, COL_DRAFT_CTX, COL_VERIFY_CTX, COL_ROWS, COL_REFRESHED = range(6)


def record_matrix(records: Iterable[IterationRecord]) -> np.ndarray:
    """[iterations, 6] int64: accepted, ngram_accepted, draft_ctx, verify_ctx,
    verify_rows, refreshed."""
    recs = list(records)
    m = np.zeros((len(recs), 6), dtype=np.int64)
    for i, r in enumerate(recs):
        m[i] = (r.accepted, r.ngram_accepted, r.draft_ctx, r.verify_ctx, r.verify_rows, int(r.refreshed))
    return m


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
        return {"iterations": self.iterations, "gamma": self.gamma, "accepted": list(self.accepted),
                "ngram_accepted": list(self.ngram_accepted), "alpha": self.alpha, "beta": self.beta,
                "emitted": self.emitted, "distinct": {str(n): v for n, v in self.distinct.items()},
                "forward_counts": dict(self.forward_counts), "wall_times": dict(self.wall_times)}


def _rate(column: np.ndarray, gamma: int) -> float:
    if column.size == 0:
        raise ValueError("acceptance rate needs at least one iteration")
    return float(column.sum()) / ((gamma + 1) * column.size)


def acceptance_rate(records: Iterable[IterationRecord], gamma: int) -> float:
    """Eq. 5: committed tokens over (gamma + 1) per iteration."""
    return _rate(record_matrix(records)[:, COL_ACCEPTED], gamma)


def ngram_acceptance_rate(records: Iterable[IterationRecord], gamma: int) -> float:
    """Eq. 7: tokens of fully accepted n-gram branches over (gamma + 1) per iteration."""
    return _rate(record_matrix(records)[:, COL_NGRAM], gamma)


def speedup(ar_cost: float, swift_cost: float) -> float:
    """Ratio of average per-token latencies (> 1 means faster)."""
    if ar_cost <= 0 or swift_cost <= 0:
        raise ValueError("latencies must be positive")
    return ar_cost / swift_cost


def distinct_n(tokens: list[int], n: int) -> float:
    """Unique n-token windows over all windows."""
    if len(tokens) < n:
        raise SequenceTooShort(f"{len(tokens)} tokens cannot form an {n}-gram")
    arr = np.asarray(tokens, dtype=np.int64)
    windows = np.lib.stride_tricks.sliding_window_view(arr, n)
    return np.unique(windows, axis=0).shape[0] / windows.shape[0]


def distinct_average(tokens: list[int], ns: tuple[int, ...] = (1, 2, 3, 4)) -> dict[int, float]:
    return {n: distinct_n(tokens, n) for n in ns if len(tokens) >= n}


def collect_metrics(records: list[IterationRecord], gamma: int, emitted_tokens: list[int],
                    forward_counts: dict[str, int] | None = None,
                    wall_times: dict[str, float] | None = None) -> RunMetrics:
    m = record_matrix(records)
    return RunMetrics(iterations=m.shape[0], gamma=gamma, accepted=m[:, COL_ACCEPTED].tolist(),
                      ngram_accepted=m[:, COL_NGRAM].tolist(), alpha=_rate(m[:, COL_ACCEPTED], gamma),
                      beta=_rate(m[:, COL_NGRAM], gamma), emitted=len(emitted_tokens),
                      distinct=distinct_average(list(emitted_tokens)), forward_counts=dict(forward_counts or {}),
                      wall_times=dict(wall_times or {}))


def write_trace(records: Iterable[IterationRecord], path: str | Path) -> None:
    """One JSON object per line (the reference's trace format)."""
    Path(path).write_text("".join(r.to_json() + "\n" for r in records), encoding="utf-8")


def read_trace(path: str | Path) -> list[IterationRecord]:
    with open(path, encoding="utf-8") as fh:
        return [IterationRecord.from_json(s) for s in (line.strip() for line in fh) if s]


# ------------------------------------------------------------ cost model --
@dataclass(frozen=True)
class CostParams:
    """Bytes and flops of one forward for the roofline replay of a trace:
    a forward costs max(bytes / bandwidth, rows * row_ops / flops), with bytes
    = weights + K/V of the attended context. Defaults are the reference's
    (A100-80G, 8B model in bf16); `B200` below is this repo's target."""

    bandwidth: float = 2.04e12
    flops: float = 312e12
    weight_bytes: float = 15.0e9
    kv_bytes_per_token: float = 131072.0
    ops_per_row: float | None = None

    def __post_init__(self) -> None:
        if min(self.bandwidth, self.flops, self.weight_bytes) <= 0:
            raise ValueError("hardware parameters must be positive")

    @property
    def row_ops(self) -> float:
        return self.weight_bytes if self.ops_per_row is None else self.ops_per_row


# one B200 (measured HBM copy bandwidth and sustained dense bf16, MEASURED_PEAKS.json of
# this pool) running the cfg3 model: 6.213e9 reference-architecture params in bf16,
# 2 flops per parameter per row
B200 = CostParams(bandwidth=6556.2e9, flops=1363.3e12, weight_bytes=12.43e9, kv_bytes_per_token=131072.0,
                  ops_per_row=2 * 6.213e9)


def load_time(num_bytes: float, bandwidth: float) -> float:
    return num_bytes / bandwidth


def compute_time(ops: float, flops: float) -> float:
    return ops / flops


def _forward_times(params: CostParams, kv_tokens: np.ndarray, rows: np.ndarray) -> np.ndarray:
    mem = (params.weight_bytes + params.kv_bytes_per_token * kv_tokens.astype(np.float64)) / params.bandwidth
    return np.maximum(mem, rows.astype(np.float64) * params.row_ops / params.flops)


def forward_time(params: CostParams, kv_tokens: int, rows: int = 1) -> float:
    return float(_forward_times(params, np.asarray([kv_tokens]), np.asarray([rows]))[0])


def ar_generation_cost(params: CostParams, prefix_len: int, gen_len: int) -> float:
    """Seconds of token-by-token decoding with the cache growing from the prompt."""
    ctx = prefix_len + np.arange(gen_len, dtype=np.int64)
    return float(_forward_times(params, ctx, np.ones_like(ctx)).sum())


def swift_generation_cost(params: CostParams, records: Iterable[IterationRecord]) -> float:
    """Seconds of a traced speculative run: per iteration one draft forward over
    the partial cache and one verification forward over the full cache."""
    m = record_matrix(records)
    if m.shape[0] == 0:
        return 0.0
    draft = _forward_times(params, m[:, COL_DRAFT_CTX], np.ones(m.shape[0], dtype=np.int64))
    verify = _forward_times(params, m[:, COL_VERIFY_CTX], np.maximum(m[:, COL_ROWS], 1))
    return float(draft.sum() + verify.sum())


def simulated_speedup(params: CostParams, records: list[IterationRecord], prefix_len: int) -> float:
    emitted = int(record_matrix(records)[:, COL_ACCEPTED].sum())
    if emitted == 0:
        raise ValueError("trace committed no tokens")
    return speedup(ar_generation_cost(params, prefix_len, emitted) / emitted,
                   swift_generation_cost(params, records) / emitted)


def forward_bytes(weight_bytes: float, kv_bytes_per_token: float, ctx: int) -> float:
    """HBM bytes of one forward streaming the weights and `ctx` tokens of K/V."""
    return weight_bytes + kv_bytes_per_token * ctx


def step_bound_seconds(params: CostParams, ctx: int, budget: int) -> float:
    """Lower bound of one decode iteration on `params`' bandwidth: a draft
    forward over `budget` partial-cache entries plus a verification forward
    over `ctx` full-cache entries (32.5 GB at cfg3 ctx 54K)."""
    return (forward_bytes(params.weight_bytes, params.kv_bytes_per_token, budget)
            + forward_bytes(params.weight_bytes, params.kv_bytes_per_token, ctx)) / params.bandwidth
