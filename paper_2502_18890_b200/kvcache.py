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
  re-sorting. The importance order (sink, then body) is a per-layer device
  ring of slot ids with a free-slot stack beside it, so admit / evict is a
  device kernel that reads the accepted count from the step result: it runs
  inside the engine's CUDA graph with no host round trip.
"""

from __future__ import annotations

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
    """Budgeted drafting cache: fixed sink + importance-ordered body, on device.

    Per layer the device holds slot metadata (pos / rank / score), the slot
    K_raw / V rows, the body's importance order as a ring of slot ids and a
    free-slot stack (include/swiftdec_b200.h, SD_PM_*). Every layer admits and
    evicts the same NUMBER of entries, so the host mirrors only the counters
    (count, hi, free count, mark); which slots move is decided on the device,
    which lets the engine run admit/evict inside its CUDA graph."""

    _BATCH = 1024  # entries moved each way per sd_partial_step launch

    def __init__(self, sink_size: int, budget: int, num_layers: int, num_kv_heads: int, head_dim: int,
                 dtype: torch.dtype = torch.bfloat16, device: str | torch.device = "cuda", slot_cap: int | None = None):
        if budget <= sink_size:
            raise BudgetTooSmall(f"budget {budget} must exceed sink size {sink_size}")
        L.require_cuda()
        self.sink_size, self.budget, self.num_layers = sink_size, budget, num_layers
        self.num_kv_heads, self.head_dim, self.dtype = num_kv_heads, head_dim, dtype
        self.device = torch.device(device)
        self.slot_cap = slot_cap or (budget + L.TREE_MAX_DEPTH)
        self._alloc(self.slot_cap)
        self.hi = 0      # slots [0, hi) scanned by the draft kernel (same on every layer)
        self.nfree = 0   # holes below hi
        self.count = 0
        self.mark = 0

    def _alloc(self, cap: int) -> None:
        Ln, Hk, dh = self.num_layers, self.num_kv_heads, self.head_dim
        self.pk = torch.zeros((Ln, Hk, cap, dh), dtype=self.dtype, device=self.device)
        self.pv = torch.zeros_like(self.pk)
        self.ppos = torch.full((Ln, cap), -1, dtype=torch.int32, device=self.device)
        self.prank = torch.full((Ln, cap), -1, dtype=torch.int32, device=self.device)
        self.pscore = torch.full((Ln, cap), float("nan"), dtype=torch.float32, device=self.device)
        self.pring = torch.zeros((Ln, cap), dtype=torch.int32, device=self.device)
        self.pfree = torch.zeros((Ln, cap), dtype=torch.int32, device=self.device)
        self.pmeta = torch.zeros((Ln, L.PM_WORDS), dtype=torch.int32, device=self.device)
        self.slot_cap = cap
        self.tmaps = None
        self._make_tmaps()

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

    def count_dev(self) -> torch.Tensor:
        """Device int32 view of layer 0's live-entry count: the draft row's
        rotation position (engine.py:202-206), read inside the step graph."""
        return self.pmeta[0, L.PM_COUNT:L.PM_COUNT + 1]

    def _slot_args(self):
        return (self.slot_cap, L.ptr(self.ppos), L.ptr(self.prank), L.ptr(self.pscore), L.ptr(self.pring),
                L.ptr(self.pfree), L.ptr(self.pmeta))

    # ---- host views (reference field names; device -> host copies) ----
    def order(self) -> list[list[int]]:
        """Per layer: slot ids in the reference's list order (sink, then body
        by importance, kvcache.py:197)."""
        meta = self.pmeta.cpu().numpy()
        ring = self.pring.cpu().numpy()
        out = []
        for l in range(self.num_layers):
            head, ln = int(meta[l, L.PM_HEAD]), int(meta[l, L.PM_LEN])
            body = [int(ring[l, (head + i) % self.slot_cap]) for i in range(ln)]
            out.append(list(range(min(self.sink_size, self.count))) + body)
        return out

    @property
    def positions(self) -> list[list[int]]:
        pos = self.ppos.cpu().numpy()
        return [[int(pos[l, s]) for s in o] for l, o in enumerate(self.order())]

    @property
    def scores(self) -> list[list[float | None]]:
        sc = self.pscore.cpu().numpy()
        return [[None if np.isnan(sc[l, s]) else float(sc[l, s]) for s in o] for l, o in enumerate(self.order())]

    @property
    def k(self) -> list[torch.Tensor]:
        return [self.pk[l][:, torch.as_tensor(o, dtype=torch.long, device=self.device)].permute(1, 0, 2)
                for l, o in enumerate(self.order())]

    @property
    def v(self) -> list[torch.Tensor]:
        return [self.pv[l][:, torch.as_tensor(o, dtype=torch.long, device=self.device)].permute(1, 0, 2)
                for l, o in enumerate(self.order())]

    def ranks(self) -> np.ndarray:
        return self.prank.cpu().numpy()

    def device_error(self) -> int:
        return int(self.pmeta[:, L.PM_ERR].max().item())

    # ---- builds (kvcache.py:268-329) ----
    def _reset_counts(self, count: int, upto: int) -> None:
        self.count = self.hi = count
        self.nfree = 0
        self.mark = upto

    def build_mirror(self, full: FullCache, upto: int) -> None:
        L.call("sd_partial_mirror", self.num_layers, self.num_kv_heads, self.head_dim, upto, self.sink_size,
               L.ptr(full.k_raw), L.ptr(full.v), L.dcode(self.dtype), full.layer_stride, full.head_stride,
               L.ptr(self.pk), L.ptr(self.pv), self.layer_stride, self.head_stride, *self._slot_args(), L.stream())
        self._reset_counts(upto, upto)

    def refresh_from(self, full: FullCache, upto: int, q_sum: torch.Tensor | None = None,
                     scores: torch.Tensor | None = None, num_heads: int | None = None) -> None:
        """Fused Eq. 2 score -> top-K -> gather (one launch): from the summed
        last queries q_sum [L, H, dh], or from precomputed scores [L, upto-sink]
        (sharded refresh, prefill_partial)."""
        n, take = upto - self.sink_size, self.budget - self.sink_size
        ws = self._refresh_ws(n, take)
        H = num_heads if num_heads is not None else (q_sum.shape[1] if q_sum is not None else self.num_kv_heads)
        L.call("sd_partial_refresh", L.ptr(q_sum), L.ptr(scores), self.num_layers, H, self.num_kv_heads,
               self.head_dim, upto, self.sink_size, self.budget, L.ptr(full.k_raw), L.ptr(full.v),
               L.dcode(self.dtype), full.layer_stride, full.head_stride, L.ptr(self.pk), L.ptr(self.pv),
               self.layer_stride, self.head_stride, *self._slot_args(), L.ptr(ws), ws.numel(), L.stream())
        self._reset_counts(self.budget, upto)

    def _refresh_ws(self, n: int, take: int) -> torch.Tensor:
        need = L.load().sd_refresh_workspace_bytes(self.num_layers, n, take)
        if getattr(self, "_ws", None) is None or self._ws.numel() < need:
            self._ws = torch.empty(int(need * 1.25) + 1024, dtype=torch.uint8, device=self.device)
        return self._ws

    def build_topk(self, full: FullCache, scores: torch.Tensor, upto: int) -> None:
        """scores: [L, upto - sink] fp32 on device."""
        self.refresh_from(full, upto, scores=scores.contiguous())

    # ---- maintenance (kvcache.py:215-225, 332-354) ----
    def _account(self, a: int, evict: bool) -> None:
        """Host mirror of the device counters after admitting a and (evict)
        trimming to the budget."""
        over = max(0, self.count + a - self.budget) if evict else 0
        self.nfree += over
        reuse = min(self.nfree, a)
        self.nfree -= reuse
        self.hi += a - reuse
        self.count += a - over

    def _step(self, full: FullCache | None, a: int, first_pos: int, evict: bool, protected: int,
              result: torch.Tensor | None = None) -> None:
        fk = L.ptr(full.k_raw) if full is not None else None
        fv = L.ptr(full.v) if full is not None else None
        fls = full.layer_stride if full is not None else 0
        fhs = full.head_stride if full is not None else 0
        L.call("sd_partial_step", self.num_layers, L.ptr(result), a, first_pos, int(evict), protected,
               self.sink_size, self.budget, self.num_kv_heads, self.head_dim, fk, fv, L.dcode(self.dtype), fls, fhs,
               L.ptr(self.pk), L.ptr(self.pv), self.layer_stride, self.head_stride, *self._slot_args(), L.stream())

    def _grow(self, need: int) -> None:
        """Reallocate the slot arrays for a burst beyond slot_cap (API path only:
        the engine admits <= 8 per step into budget + 8 slots and never grows, so
        pointers captured in its CUDA graph stay valid). Rings are re-linearised."""
        cap = max(need, 2 * self.slot_cap)
        old = (self.pk, self.pv, self.ppos, self.prank, self.pscore)
        meta = self.pmeta.clone()
        ring = self.pring.cpu().numpy()
        free = self.pfree.clone()
        oc = self.slot_cap
        self._alloc(cap)
        self.pk[:, :, :oc], self.pv[:, :, :oc] = old[0], old[1]
        self.ppos[:, :oc], self.prank[:, :oc], self.pscore[:, :oc] = old[2], old[3], old[4]
        self.pfree[:, :oc] = free
        m = meta.cpu().numpy()
        lin = np.zeros((self.num_layers, cap), dtype=np.int32)
        for l in range(self.num_layers):
            head, ln = int(m[l, L.PM_HEAD]), int(m[l, L.PM_LEN])
            lin[l, :ln] = [ring[l, (head + i) % oc] for i in range(ln)]
        self.pring.copy_(torch.as_tensor(lin))
        meta[:, L.PM_HEAD] = 0
        self.pmeta.copy_(meta)

    def admit(self, positions, full: FullCache) -> None:
        """Copy newly committed consecutive positions to the body head."""
        positions = [int(p) for p in positions]
        if not positions:
            return
        if positions != list(range(positions[0], positions[0] + len(positions))):
            raise ValueError("admitted positions must be consecutive")
        if self.hi + len(positions) - self.nfree > self.slot_cap:
            self._grow(self.hi + len(positions) - self.nfree)
        for i in range(0, len(positions), self._BATCH):
            a = min(self._BATCH, len(positions) - i)
            self._step(full, a, positions[i], False, 0)
            self._account(a, False)

    def evict(self, protected: int = 0) -> None:
        over = self.count - self.budget
        if over <= 0:
            return
        if self.count - self.sink_size - over < protected:
            raise SinkViolation("eviction would reach protected entries; body capacity "
                                f"{self.capacity} is smaller than one iteration's acceptance")
        while self.count > self.budget:
            b = min(self._BATCH, self.count - self.budget)
            L.call("sd_partial_step", self.num_layers, None, 0, 0, 1, 0, self.sink_size, self.count - b,
                   self.num_kv_heads, self.head_dim, None, None, L.dcode(self.dtype), 0, 0, L.ptr(self.pk),
                   L.ptr(self.pv), self.layer_stride, self.head_stride, *self._slot_args(), L.stream())
            self.nfree += b
            self.count -= b

    def admit_evict(self, first_pos: int, a: int, full: FullCache, protected: int) -> None:
        """Engine path (eager): admit a consecutive positions and trim to budget in one launch."""
        over = self.count + a - self.budget
        if over > 0 and self.count + a - self.sink_size - over < protected:
            raise SinkViolation("eviction would reach protected entries; body capacity "
                                f"{self.capacity} is smaller than one iteration's acceptance")
        if self.hi + a - min(self.nfree + max(over, 0), a) > self.slot_cap:
            raise ValueError("admit_evict beyond the slot capacity")
        self._step(full, a, first_pos, True, protected)
        self._account(a, True)

    def step_device(self, full: FullCache, result: torch.Tensor) -> None:
        """Engine path inside the CUDA graph: a and the first position come from
        the device step result (engine.py:281-283); call account() on the host
        once the accepted count is known."""
        self._step(full, -1, 0, True, 0, result=result)

    def account(self, a: int) -> None:
        self._account(a, True)

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
