"""Contextual-penalty sampling on device (API mirror of swiftdec/sampling.py).

p_i = exp(l_i / (t * I_i)) / Z with I_i = theta for tokens in the recent
window (sampling.py:142-162), top-p / min-p / eta truncation
(sampling.py:193-216) and an inverse-CDF draw at the (seed, position) deviate
(sampling.py:219-224). All arithmetic runs in fp64 inside `sd_sample_rows`
(csrc/sampling.cu); the window is a device ring plus a per-token count array.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L


@dataclass(frozen=True)
class Truncation:
    kind: str
    value: float
    eta_alpha: float | None = None

    def __post_init__(self) -> None:
        if self.kind not in ("top_p", "min_p", "eta"):
            raise ValueError(f"unknown truncation kind: {self.kind}")
        if not (0.0 < self.value <= 1.0):
            raise ValueError(f"truncation parameter must be in (0, 1], got {self.value}")

    @classmethod
    def top_p(cls, p: float) -> "Truncation":
        return cls("top_p", p)

    @classmethod
    def min_p(cls, p_base: float) -> "Truncation":
        return cls("min_p", p_base)

    @classmethod
    def eta(cls, eps: float, alpha: float | None = None) -> "Truncation":
        return cls("eta", eps, alpha)

    @property
    def code(self) -> int:
        return {"top_p": L.TRUNC_TOP_P, "min_p": L.TRUNC_MIN_P, "eta": L.TRUNC_ETA}[self.kind]


@dataclass(frozen=True)
class SamplerConfig:
    temperature: float = 1.0
    theta: float = 1.2
    window: int = 1024
    truncation: Truncation = field(default_factory=lambda: Truncation.min_p(0.1))
    seed: int = 0
    ctrl_style: bool = False

    def __post_init__(self) -> None:
        if self.temperature <= 0.0:
            raise ValueError("temperature must be > 0")
        if self.theta < 1.0:
            raise ValueError("theta must be >= 1.0")
        if self.window < 0:
            raise ValueError("window must be >= 0")


class PenaltyWindow:
    """Device ring of the last `capacity` generated tokens + per-token counts.

    `state` is the session state vector (int64[16]); slots ST_RING_HEAD /
    ST_RING_LEN hold the ring head and length, updated by device kernels.
    """

    def __init__(self, capacity: int, vocab_size: int, state: torch.Tensor | None = None,
                 device: str | torch.device = "cuda"):
        L.require_cuda()
        self.capacity, self.vocab_size = capacity, vocab_size
        self.device = torch.device(device)
        self.ring = torch.zeros(max(1, capacity), dtype=torch.int32, device=self.device)
        self.count = torch.zeros(vocab_size, dtype=torch.int32, device=self.device)
        self.state = state if state is not None else torch.zeros(16, dtype=torch.int64, device=self.device)
        self.host_len = 0  # mirrored on the host by whoever pushes

    def __len__(self) -> int:
        return int(self.state[L.ST_RING_LEN].item())

    def __contains__(self, token: int) -> bool:
        return bool(self.count[int(token)].item() > 0)

    def push(self, token: int) -> None:
        self.push_many([token])

    def push_many(self, tokens) -> None:
        toks = [int(t) for t in tokens]
        if not toks or self.capacity == 0:
            return
        t = torch.tensor(toks, dtype=torch.int32, device=self.device)
        L.call("sd_window_push", L.ptr(t), len(toks), L.ptr(self.state), L.ptr(self.ring), L.ptr(self.count),
               self.capacity, L.stream())
        self.host_len = min(self.capacity, self.host_len + len(toks))

    def members(self) -> set[int]:
        return set(torch.nonzero(self.count > 0).flatten().tolist())

    def member_mask(self) -> np.ndarray:
        return (self.count > 0).cpu().numpy()

    def ring_tokens(self) -> list[int]:
        """Ring contents, oldest first."""
        head, n = int(self.state[L.ST_RING_HEAD].item()), len(self)
        r = self.ring.cpu().tolist()
        return [r[(head + i) % self.capacity] for i in range(n)]

    def shrunk_masks(self, max_drop: int) -> list[np.ndarray]:
        """masks[j] = membership with the j oldest ring entries removed (sampling.py:120-139)."""
        cnt = self.count.cpu().numpy().astype(np.int64)
        masks = [cnt > 0]
        for old in self.ring_tokens()[: min(max_drop, len(self))]:
            cnt[old] -= 1
            masks.append(cnt > 0)
        while len(masks) <= max_drop:
            masks.append(masks[-1])
        return masks


def _as_dev(x, dtype=torch.float64) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(x), dtype=dtype, device="cuda").contiguous()


def _args(rows, V, in_kind, cfg_t=1.0, theta=1.0, ctrl=False, member_kind=L.MEMBER_NONE, mask=None,
          trunc=None, seed=0, positions=None):
    a = L.SampleArgs()
    a.rows, a.V, a.in_kind = rows, V, in_kind
    a.temperature, a.theta, a.ctrl_style = float(cfg_t), float(theta), int(bool(ctrl))
    a.member_kind = member_kind
    a.member_mask = L.ptr(mask)
    a.window, a.depth = 0, 1
    a.trunc_kind = trunc.code if trunc is not None else L.TRUNC_NONE
    a.trunc_value = float(trunc.value) if trunc is not None else 0.0
    a.eta_alpha = float(trunc.eta_alpha) if (trunc is not None and trunc.eta_alpha is not None) else -1.0
    a.seed = seed & ((1 << 64) - 1)
    a.positions = L.ptr(positions)
    return a


def penalized_probs_masked(logits, member_mask, config: SamplerConfig) -> torch.Tensor:
    """Penalised softmax with an explicit membership mask; (..., V) -> fp64 (device)."""
    lg = _as_dev(logits)
    shape = lg.shape
    lg2 = lg.reshape(-1, shape[-1])
    rows, V = lg2.shape
    mk = torch.as_tensor(np.broadcast_to(np.asarray(member_mask if not isinstance(member_mask, torch.Tensor)
                                                    else member_mask.cpu().numpy(), dtype=bool), shape),
                         device="cuda").reshape(rows, V).to(torch.uint8).contiguous()
    out = torch.empty((rows, V), dtype=torch.float64, device="cuda")
    pos = torch.zeros(rows, dtype=torch.int32, device="cuda")
    a = _args(rows, V, L.IN_LOGITS_F64, config.temperature, config.theta, config.ctrl_style, L.MEMBER_MASK, mk,
              positions=pos)
    a.probs_out = L.ptr(out)
    L.call("sd_sample_rows", L.ptr(lg2), a, L.stream())
    return out.reshape(shape)


def penalized_probs(logits, window: PenaltyWindow, config: SamplerConfig) -> torch.Tensor:
    return penalized_probs_masked(logits, window.member_mask(), config)


def truncate(dist, rule: Truncation) -> torch.Tensor:
    d = _as_dev(dist)
    V = d.shape[-1]
    d2 = d.reshape(-1, V)
    out = torch.empty_like(d2)
    pos = torch.zeros(d2.shape[0], dtype=torch.int32, device="cuda")
    a = _args(d2.shape[0], V, L.IN_PROBS_F64, trunc=rule, positions=pos)
    a.trunc_out = L.ptr(out)
    L.call("sd_sample_rows", L.ptr(d2), a, L.stream())
    return out.reshape(d.shape)


def sample_at(dist, position: int, seed: int) -> int:
    d = _as_dev(dist).reshape(1, -1)
    pos = torch.tensor([int(position)], dtype=torch.int32, device="cuda")
    tok = torch.empty(1, dtype=torch.int32, device="cuda")
    a = _args(1, d.shape[1], L.IN_PROBS_F64, seed=seed, positions=pos)
    a.token_out = L.ptr(tok)
    L.call("sd_sample_rows", L.ptr(d), a, L.stream())
    return int(tok.item())


def softmax(scaled) -> torch.Tensor:
    return penalized_probs_masked(scaled, np.zeros(np.shape(scaled)[-1], dtype=bool),
                                  SamplerConfig(temperature=1.0, theta=1.0, window=0))


def entropy(dist) -> float:
    p = np.asarray(dist.cpu() if isinstance(dist, torch.Tensor) else dist, dtype=np.float64)
    p = p[p > 0.0]
    return float(-np.sum(p * np.log(p)))


def eta_threshold(rule: Truncation, dist) -> float:
    alpha = rule.eta_alpha if rule.eta_alpha is not None else math.sqrt(rule.value)
    return min(rule.value, alpha * math.exp(-entropy(dist)))
