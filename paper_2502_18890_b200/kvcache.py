"""Device KV caches (API mirror of swiftdec/kvcache.py).

HBM layout (per session, allocated once):

* FullCache: K_raw, K_rot, V as [L][Hk][cap][dh] (dtype) — one kv head's rows
  are contiguous, so split-KV attention streams each head linearly and a
  KV-head shard is a plain slice. Rows beyond the committed length hold
  staged tree rows of the current verification (kvcache.py:84-96).
* PartialCache: K_raw, V as [L][Hk][slot_cap][dh] plus per-layer slot
  metadata pos / rank / score ([L][slot_cap]). Ranks are the position order
  of the live slots, maintained incrementally on admit / evict, so the draft
  kernel rotates K_raw at its rank on load (kvcache.py:136-165) without ever
  re-sorting. The importance order (sink, then body) is a host-side deque of
  slot ids shared by all layers: every layer admits and evicts the same
  number of entries at the same slot ids, only the slot contents differ.
"""

from __future__ import annotations

from collections import deque

import numpy as np
import torch

from . import _lib as L


class GroupMismatch(ValueError):
    """Query head count is not group_size times the KV head count."""


class BudgetTooSmall(ValueError):
    """Cache budget does not exceed the sink size."""


class SinkViolation(RuntimeError):
    """Eviction would reach the sink or a just-admitted entry."""


class CapacityExceeded(RuntimeError):
    """The preallocated device cache is full."""


class FullCache:
    """Append-only device K/V store of the committed sequence."""

    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, capacity: int = 4096,
                 dtype: torch.dtype = torch.bfloat16, device: str | torch.device = "cuda"):
        L.require_cuda()
        self.num_layers, self.num_kv_heads, self.head_dim = num_layers, num_kv_heads, head_dim
        self.capacity, self.dtype, self.device = capacity, dtype, torch.device(device)
        shape = (num_layers, num_kv_heads, capacity, head_dim)
        self.k_raw = torch.zeros(shape, dtype=dtype, device=self.device)
        self.k_rot = torch.zeros(shape, dtype=dtype, device=self.device)
        self.v = torch.zeros(shape, dtype=dtype, device=self.device)
        self.positions: list[int] = []
        self.tmaps = None
        if dtype == torch.bfloat16 and head_dim == 128:
            # TMA descriptors for the tensor-core verification path (sd_attention)
            import ctypes
            tk, tv = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
            L.call("sd_make_kv_tmap", L.ptr(self.k_rot), num_layers, num_kv_heads, capacity, head_dim, tk)
            L.call("sd_make_kv_tmap", L.ptr(self.v), num_layers, num_kv_heads, capacity, head_dim, tv)
            self.tmaps = (tk, tv)

    # strides in elements
    @property
    def head_stride(self) -> int:
        return self.capacity * self.head_dim

    @property
    def layer_stride(self) -> int:
        return self.num_kv_heads * self.capacity * self.head_dim

    def __len__(self) -> int:
        return len(self.positions)

    def reserve(self, extra: int) -> None:
        if len(self) + extra > self.capacity:
            raise CapacityExceeded(f"full cache capacity {self.capacity} < {len(self) + extra}")

    def stage(self, layer: int, offset: int, k_raw, k_rot, v) -> None:
        i = len(self) + offset
        self.k_raw[layer, :, i] = torch.as_tensor(np.asarray(k_raw), dtype=self.dtype, device=self.device)
        self.k_rot[layer, :, i] = torch.as_tensor(np.asarray(k_rot), dtype=self.dtype, device=self.device)
        self.v[layer, :, i] = torch.as_tensor(np.asarray(v), dtype=self.dtype, device=self.device)

    def commit_rows(self, positions) -> None:
        self.positions.extend(int(p) for p in positions)

    def ensure_rotated(self, rope=None) -> None:
        pass

    def raw_keys(self, layer: int, upto: int) -> torch.Tensor:
        return self.k_raw[layer, :, :upto].permute(1, 0, 2)

    def rotated_keys(self, layer: int, upto: int) -> torch.Tensor:
        return self.k_rot[layer, :, :upto].permute(1, 0, 2)

    def values(self, layer: int, upto: int) -> torch.Tensor:
        return self.v[layer, :, :upto].permute(1, 0, 2)

    def truncate(self, n: int) -> None:
        del self.positions[n:]

    def reconcile_device(self, base_len: int, result: torch.Tensor, q_pre=None, q_rows=0, num_heads=0,
                         q_sum=None) -> None:
        """Compact kept rows (keep offsets from the device step result)."""
        L.call("sd_reconcile", self.num_layers, L.ptr(result), base_len, L.ptr(self.k_raw), L.ptr(self.k_rot),
               L.ptr(self.v), L.dcode(self.dtype), self.layer_stride, self.head_stride, self.num_kv_heads,
               self.head_dim, L.ptr(q_pre), q_rows, num_heads, L.ptr(q_sum), L.stream())

    def reconcile(self, base_len: int, keep_offsets) -> None:
        """kvcache.py:116-127."""
        keep = [int(k) for k in keep_offsets]
        res = torch.full((32,), -1, dtype=torch.int32)
        res[L.RES_ACCEPTED] = len(keep)
        res[L.RES_KEEP:L.RES_KEEP + len(keep)] = torch.tensor(keep, dtype=torch.int32)
        self.reconcile_device(base_len, res.to(self.device))
        self.positions = self.positions[:base_len] + [self.positions[base_len + k] for k in keep]

    def gather(self, layer: int, positions):
        idx = torch.as_tensor(list(positions), dtype=torch.long, device=self.device)
        return (self.k_raw[layer, :, idx].permute(1, 0, 2).clone(), self.v[layer, :, idx].permute(1, 0, 2).clone())


class PartialCache:
    """Budgeted drafting cache: fixed sink + importance-ordered body, on device."""

    def __init__(self, sink_size: int, budget: int, num_layers: int, num_kv_heads: int, head_dim: int,
                 dtype: torch.dtype = torch.bfloat16, device: str | torch.device = "cuda", slot_cap: int | None = None):
        if budget <= sink_size:
            raise BudgetTooSmall(f"budget {budget} must exceed sink size {sink_size}")
        L.require_cuda()
        self.sink_size, self.budget, self.num_layers = sink_size, budget, num_layers
        self.num_kv_heads, self.head_dim, self.dtype = num_kv_heads, head_dim, dtype
        self.device = torch.device(device)
        self.slot_cap = slot_cap or (budget + L.TREE_MAX_DEPTH)
        shape = (num_layers, num_kv_heads, self.slot_cap, head_dim)
        self.pk = torch.zeros(shape, dtype=dtype, device=self.device)
        self.pv = torch.zeros(shape, dtype=dtype, device=self.device)
        self.ppos = torch.full((num_layers, self.slot_cap), -1, dtype=torch.int32, device=self.device)
        self.prank = torch.full((num_layers, self.slot_cap), -1, dtype=torch.int32, device=self.device)
        self.pscore = torch.full((num_layers, self.slot_cap), float("nan"), dtype=torch.float32, device=self.device)
        self.tmaps = None
        self._make_tmaps()
        self.body: deque[int] = deque()  # slot ids in importance order (shared by all layers)
        self.free: list[int] = []        # holes below `hi`
        self.hi = 0                      # slots [0, hi) scanned by the draft kernel
        self.count = 0
        self.mark = 0

    def _make_tmaps(self) -> None:
        # TMA descriptors (64-slot boxes) for the tensor-core draft attention
        if self.dtype == torch.bfloat16 and self.head_dim == 128:
            import ctypes
            tk, tv = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
            L.call("sd_make_slot_tmap", L.ptr(self.pk), self.num_layers, self.num_kv_heads, self.slot_cap,
                   self.head_dim, tk)
            L.call("sd_make_slot_tmap", L.ptr(self.pv), self.num_layers, self.num_kv_heads, self.slot_cap,
                   self.head_dim, tv)
            self.tmaps = (tk, tv)

    @property
    def head_stride(self) -> int:
        return self.slot_cap * self.head_dim

    @property
    def layer_stride(self) -> int:
        return self.num_kv_heads * self.slot_cap * self.head_dim

    @property
    def capacity(self) -> int:
        return self.budget - self.sink_size

    def __len__(self) -> int:
        return self.count

    # ---- host views (reference field names; device -> host copies) ----
    def order(self) -> list[int]:
        return list(range(min(self.sink_size, self.count))) + list(self.body)

    @property
    def positions(self) -> list[list[int]]:
        pos = self.ppos.cpu().numpy()
        o = self.order()
        return [[int(pos[l, s]) for s in o] for l in range(self.num_layers)]

    @property
    def scores(self) -> list[list[float | None]]:
        sc = self.pscore.cpu().numpy()
        o = self.order()
        return [[None if np.isnan(sc[l, s]) else float(sc[l, s]) for s in o] for l in range(self.num_layers)]

    @property
    def k(self) -> list[torch.Tensor]:
        idx = torch.as_tensor(self.order(), dtype=torch.long, device=self.device)
        return [self.pk[l][:, idx].permute(1, 0, 2) for l in range(self.num_layers)]

    @property
    def v(self) -> list[torch.Tensor]:
        idx = torch.as_tensor(self.order(), dtype=torch.long, device=self.device)
        return [self.pv[l][:, idx].permute(1, 0, 2) for l in range(self.num_layers)]

    def ranks(self) -> np.ndarray:
        return self.prank.cpu().numpy()

    # ---- builds (kvcache.py:268-319) ----
    def _reset_slots(self, count: int) -> None:
        self.count = count
        self.hi = count
        self.free = []
        self.body = deque(range(self.sink_size, count))

    def build_mirror(self, full: FullCache, upto: int) -> None:
        L.call("sd_mirror_positions", self.num_layers, upto, self.sink_size, L.ptr(self.ppos), L.ptr(self.prank),
               L.ptr(self.pscore), self.slot_cap, L.stream())
        self._reset_slots(upto)
        self._gather(full)
        self.mark = upto

    def build_topk(self, full: FullCache, scores: torch.Tensor, upto: int) -> None:
        """scores: [L, upto - sink] fp32 on device."""
        take = self.budget - self.sink_size
        n = upto - self.sink_size
        ws = torch.empty(L.load().sd_select_workspace_bytes(self.num_layers, n), dtype=torch.uint8,
                         device=self.device)
        L.call("sd_select_topk", L.ptr(scores), self.num_layers, n, self.sink_size, take, L.ptr(self.ppos),
               L.ptr(self.prank), L.ptr(self.pscore), self.slot_cap, L.ptr(ws), ws.numel(), L.stream())
        self._reset_slots(self.budget)
        self._gather(full)
        self.mark = upto

    def _gather(self, full: FullCache) -> None:
        L.call("sd_gather_slots", self.num_layers, self.count, L.ptr(self.ppos), self.slot_cap, L.ptr(full.k_raw),
               L.ptr(full.v), L.dcode(self.dtype), full.layer_stride, full.head_stride, L.ptr(self.pk),
               L.ptr(self.pv), self.layer_stride, self.head_stride, self.num_kv_heads, self.head_dim, L.stream())

    # ---- maintenance (kvcache.py:215-225, 332-354) ----
    # One sd_partial_update launch moves at most SD_TREE_MAX_DEPTH (8) entries
    # each way; larger admit / evict bursts are split into launches of <= 8
    # (evictions first, then admissions in position order), which is the same
    # final state as one launch. All checks run before any host state changes.
    _BATCH = L.TREE_MAX_DEPTH

    def _launch(self, full: FullCache | None, first_pos: int, new_slots: list[int], evicted: list[int],
                count_before: int) -> None:
        B = self._BATCH
        cnt = count_before
        for i in range(0, len(evicted), B):
            gone = evicted[i:i + B]
            cnt -= len(gone)
            L.call("sd_partial_update", self.num_layers, self.hi, cnt, 0, 0, L.host_i32([]), len(gone),
                   L.host_i32(gone), L.ptr(self.ppos), L.ptr(self.prank), L.ptr(self.pscore), self.slot_cap, None,
                   None, L.dcode(self.dtype), 0, 0, None, None, self.layer_stride, self.head_stride,
                   self.num_kv_heads, self.head_dim, L.stream())
        for i in range(0, len(new_slots), B):
            new = new_slots[i:i + B]
            cnt += len(new)
            L.call("sd_partial_update", self.num_layers, self.hi, cnt, first_pos + i, len(new), L.host_i32(new), 0,
                   L.host_i32([]), L.ptr(self.ppos), L.ptr(self.prank), L.ptr(self.pscore), self.slot_cap,
                   L.ptr(full.k_raw), L.ptr(full.v), L.dcode(self.dtype), full.layer_stride, full.head_stride,
                   L.ptr(self.pk), L.ptr(self.pv), self.layer_stride, self.head_stride, self.num_kv_heads,
                   self.head_dim, L.stream())

    def _launch_update(self, full: FullCache, first_pos: int, new_slots: list[int], evicted: list[int]) -> None:
        """Engine path (<= 8 each way): evict + admit in one launch."""
        L.call("sd_partial_update", self.num_layers, self.hi, self.count, first_pos, len(new_slots),
               L.host_i32(new_slots), len(evicted), L.host_i32(evicted), L.ptr(self.ppos), L.ptr(self.prank),
               L.ptr(self.pscore), self.slot_cap, L.ptr(full.k_raw), L.ptr(full.v), L.dcode(self.dtype),
               full.layer_stride, full.head_stride, L.ptr(self.pk), L.ptr(self.pv), self.layer_stride,
               self.head_stride, self.num_kv_heads, self.head_dim, L.stream())

    def _grow(self, need: int) -> None:
        """Reallocate the slot arrays for a burst beyond slot_cap (API path only:
        the engine admits <= 8 per step into budget + 8 slots and never grows, so
        pointers captured in its CUDA graph stay valid)."""
        cap = max(need, 2 * self.slot_cap)
        L_, Hk, dh = self.num_layers, self.num_kv_heads, self.head_dim
        pk = torch.zeros((L_, Hk, cap, dh), dtype=self.dtype, device=self.device)
        pv = torch.zeros_like(pk)
        pk[:, :, :self.slot_cap] = self.pk
        pv[:, :, :self.slot_cap] = self.pv
        meta = []
        for t, fill in ((self.ppos, -1), (self.prank, -1), (self.pscore, float("nan"))):
            n = torch.full((L_, cap), fill, dtype=t.dtype, device=self.device)
            n[:, :self.slot_cap] = t
            meta.append(n)
        self.pk, self.pv = pk, pv
        self.ppos, self.prank, self.pscore = meta
        self.slot_cap = cap
        self._make_tmaps()

    def _take_slots(self, a: int) -> list[int]:
        short = a - len(self.free) - (self.slot_cap - self.hi)
        if short > 0:
            self._grow(self.slot_cap + short)
        out = []
        for _ in range(a):
            if self.free:
                out.append(self.free.pop())
            else:
                out.append(self.hi)
                self.hi += 1
        return out

    def admit(self, positions, full: FullCache) -> None:
        """Copy newly committed consecutive positions to the body head."""
        positions = [int(p) for p in positions]
        if not positions:
            return
        if positions != list(range(positions[0], positions[0] + len(positions))):
            raise ValueError("admitted positions must be consecutive")
        before = self.count
        slots = self._take_slots(len(positions))
        self.count += len(slots)
        self._launch(full, positions[0], slots, [], before)
        self.body.extendleft(reversed(slots))

    def evict(self, protected: int = 0) -> None:
        over = self.count - self.budget
        if over <= 0:
            return
        if self.count - self.sink_size - over < protected:
            raise SinkViolation("eviction would reach protected entries; body capacity "
                                f"{self.capacity} is smaller than one iteration's acceptance")
        before = self.count
        gone = [self.body.pop() for _ in range(over)]
        self.count -= over
        self._launch(None, 0, [], gone, before)
        self.free.extend(gone)

    def admit_evict(self, first_pos: int, a: int, full: FullCache, protected: int) -> None:
        """Engine path: admit a consecutive positions and trim to budget in one launch."""
        over = self.count + a - self.budget
        if over > 0 and self.count + a - self.sink_size - over < protected:
            raise SinkViolation("eviction would reach protected entries; body capacity "
                                f"{self.capacity} is smaller than one iteration's acceptance")
        if a > self._BATCH or max(over, 0) > self._BATCH:
            raise ValueError(f"admit_evict moves at most {self._BATCH} entries each way per step")
        gone = [self.body.pop() for _ in range(over)] if over > 0 else []
        self.free.extend(gone)
        slots = self._take_slots(a)
        self.count += a - len(gone)
        self._launch_update(full, first_pos, slots, gone)
        self.body.extendleft(reversed(slots))

    def draft_view(self, before_pos: int) -> "DraftView":
        return DraftView(self, before_pos)


class DraftView:
    """Drafting view of a partial cache (kvcache.py:227-240): every live entry
    with position < before_pos, rotated at its rank. In the engine all live
    entries qualify (they are committed before the pending token)."""

    def __init__(self, partial: PartialCache, before_pos: int):
        self.partial = partial
        self.before_pos = before_pos

    def __len__(self) -> int:
        return self.partial.count


def importance_scores(queries, keys, group_size: int):
    """Eq. 2 on device: score_n = sum_k sum_g q[k*G+g] . K[n, k] (kvcache.py:243-265)."""
    L.require_cuda()
    q = torch.as_tensor(np.asarray(queries) if not isinstance(queries, torch.Tensor) else queries,
                        dtype=torch.float32, device="cuda")
    k = torch.as_tensor(np.asarray(keys) if not isinstance(keys, torch.Tensor) else keys, device="cuda")
    single = k.dim() == 2
    if single:
        k = k[None]
    H, dh = q.shape
    n, Hk, _ = k.shape
    if H != group_size * Hk:
        raise GroupMismatch(f"{H} query heads cannot be partitioned into groups of {group_size} over {Hk} KV heads")
    kdt = torch.bfloat16 if k.dtype == torch.bfloat16 else torch.float32
    kt = k.to(kdt).permute(1, 0, 2).contiguous()  # [Hk, n, dh]
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    L.call("sd_importance_scores", L.ptr(q.contiguous()), L.ptr(kt), L.dcode(kdt), 0, n * dh, 1, H, Hk, dh, 0, n,
           L.ptr(out), None, L.stream())
    return out[0] if single else out


def layer_scores(full: FullCache, q_sum: torch.Tensor, num_heads: int, start: int, end: int,
                 per_head: torch.Tensor | None = None) -> torch.Tensor:
    """Per-layer Eq. 2 scores over full-cache rows [start, end) (engine.py:128-136)."""
    out = torch.empty((full.num_layers, end - start), dtype=torch.float32, device=full.device)
    L.call("sd_importance_scores", L.ptr(q_sum), L.ptr(full.k_raw), L.dcode(full.dtype), full.layer_stride,
           full.head_stride, full.num_layers, num_heads, full.num_kv_heads, full.head_dim, start, end,
           L.ptr(out), L.ptr(per_head), L.stream())
    return out


def prefill_partial(full: FullCache, sink_size: int, budget: int, scores, upto: int | None = None) -> PartialCache:
    n = len(full) if upto is None else upto
    if budget <= sink_size:
        raise BudgetTooSmall(f"budget {budget} must exceed sink size {sink_size}")
    if n < budget:
        raise ValueError(f"prefill_partial needs at least {budget} entries, have {n}")
    sc = torch.as_tensor(np.asarray(scores) if not isinstance(scores, torch.Tensor) else scores,
                         dtype=torch.float32, device=full.device).contiguous()
    part = PartialCache(sink_size, budget, full.num_layers, full.num_kv_heads, full.head_dim, full.dtype, full.device)
    part.build_topk(full, sc, n)
    return part


def mirror_partial(full: FullCache, sink_size: int, budget: int, upto: int | None = None) -> PartialCache:
    n = len(full) if upto is None else upto
    part = PartialCache(sink_size, budget, full.num_layers, full.num_kv_heads, full.head_dim, full.dtype, full.device,
                        slot_cap=max(budget, n) + L.TREE_MAX_DEPTH)
    part.build_mirror(full, n)
    return part


def needs_refresh(full_len: int, partial: PartialCache) -> bool:
    return (full_len - partial.mark) > partial.capacity


def refresh(full: FullCache, partial: PartialCache, scores) -> PartialCache:
    return prefill_partial(full, partial.sink_size, partial.budget, scores)


def evict_to_budget(partial: PartialCache, protected: int = 0) -> PartialCache:
    partial.evict(protected)
    return partial
