"""B200 TinyTransformer backend (API mirror of swiftdec/model.py).

Architecture (model.py:150-313): pre-norm rotary GQA transformer, tied
embedding / LM head, non-gated SiLU MLP of width 4d, gamma residually chained
draft heads (Eq. 1, model.py:104-120). Weights live in HBM in `dtype`
(bf16 by default, fp32 for tight parity runs); the residual stream, RMSNorm
and every GEMM accumulator are fp32.

Per layer the forward is: fused residual-add + RMSNorm (sd_add_rmsnorm) ->
QKV GEMM -> RoPE + KV staging (sd_rope_stage) -> split-KV attention
(sd_attention: verify tree / draft / AR / prefill block) -> O GEMM -> add +
RMSNorm -> W1 GEMM + SiLU -> W2 GEMM. Decode rows (<= 128) use the
weight-streaming tcgen05 GEMM (sd_gemm, N-tiled weight copies, split-K slices
summed by the consuming norm / RoPE kernel); prefill and fp32 builds use cuBLAS.

KV-head sharding (world > 1): rank r owns kv heads [r*Hk/P, (r+1)*Hk/P) and
their query heads; attention outputs are all-gathered before the replicated
O projection (parallel.py).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

import torch

from . import _lib as L
from .kvcache import DraftView, FullCache, PartialCache


class PositionOverflow(ValueError):
    """A requested position is at or beyond max_positions."""


class MaskShapeMismatch(ValueError):
    """Attention mask dimensions disagree with inputs plus cache length."""


class DimensionMismatch(ValueError):
    """Draft head weight shapes are incompatible with the hidden size."""


@dataclass(frozen=True)
class ModelConfig:
    vocab_size: int
    num_layers: int = 2
    hidden_dim: int = 64
    num_heads: int = 4
    num_kv_heads: int = 4
    gamma: int = 3
    max_positions: int = 65536
    init_seed: int = 0

    def __post_init__(self) -> None:
        if self.vocab_size <= 0 or self.num_layers <= 0 or self.hidden_dim <= 0:
            raise ValueError("vocab_size, num_layers and hidden_dim must be positive")
        if self.num_heads <= 0 or self.num_kv_heads <= 0 or self.max_positions <= 0:
            raise ValueError("head counts and max_positions must be positive")
        if self.gamma < 0:
            raise ValueError("gamma must be >= 0")
        if self.num_heads % self.num_kv_heads != 0:
            raise ValueError("num_heads must be a multiple of num_kv_heads")
        if self.hidden_dim % self.num_heads != 0:
            raise ValueError("hidden_dim must be a multiple of num_heads")
        if (self.hidden_dim // self.num_heads) % 2 != 0:
            raise ValueError("head dimension must be even for rotary encoding")

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.num_heads

    @property
    def group_size(self) -> int:
        return self.num_heads // self.num_kv_heads

    def param_count(self) -> int:
        return sum(int(np.prod(s)) for _, s, _ in param_specs(self))


@dataclass
class ForwardRequest:
    tokens: list[int]
    positions: list[int]
    cache: object
    attention_mask: np.ndarray | None = None
    heads_needed: int | None = None


@dataclass
class ForwardResult:
    bundles: torch.Tensor  # (T, gamma + 1, V) fp32, -inf for heads not computed
    queries: torch.Tensor  # (T, L, H, dh) fp32, pre-rotation


def param_specs(c: ModelConfig):
    """Reference parameter order and init scales (model.py:173-193)."""
    d, H, Hk, dh = c.hidden_dim, c.num_heads, c.num_kv_heads, c.head_dim
    specs = [("embed", (c.vocab_size, d), 0.3)]
    for i in range(c.num_layers):
        specs += [
            (f"l{i}.ln1", (d,), 0.0), (f"l{i}.wq", (d, H * dh), d ** -0.5),
            (f"l{i}.wk", (d, Hk * dh), d ** -0.5), (f"l{i}.wv", (d, Hk * dh), d ** -0.5),
            (f"l{i}.wo", (H * dh, d), (H * dh) ** -0.5), (f"l{i}.ln2", (d,), 0.0),
            (f"l{i}.w1", (d, 4 * d), d ** -0.5), (f"l{i}.w2", (4 * d, d), (4 * d) ** -0.5),
        ]
    specs.append(("ln_f", (d,), 0.0))
    specs += [(f"head{i + 1}", (d, d), 0.3 * d ** -0.5) for i in range(c.gamma)]
    return specs


def reference_tensor(c: ModelConfig, idx: int, shape, scale) -> np.ndarray:
    """One parameter from the reference's named seeded stream (model.py:195-205)."""
    if scale == 0.0:
        return np.ones(shape)
    g = np.random.default_rng(np.random.SeedSequence(entropy=c.init_seed, spawn_key=(idx,)))
    return g.normal(0.0, scale, size=shape)


def chained_draft_logits(h0, head_mats, lm_head) -> torch.Tensor:
    """Eq. 1 on device: h_i = h_{i-1} f_i + h_{i-1}; l_i = E h_i (model.py:104-120)."""
    h = torch.as_tensor(np.asarray(h0) if not isinstance(h0, torch.Tensor) else h0, dtype=torch.float64,
                        device="cuda")
    E = torch.as_tensor(np.asarray(lm_head) if not isinstance(lm_head, torch.Tensor) else lm_head,
                        dtype=torch.float64, device="cuda")
    d = h.shape[-1]
    if E.dim() != 2 or E.shape[1] != d:
        raise DimensionMismatch(f"lm_head must be (vocab, {d}), got {tuple(E.shape)}")
    hs = [h]
    for i, f in enumerate(head_mats):
        F = torch.as_tensor(np.asarray(f) if not isinstance(f, torch.Tensor) else f, dtype=torch.float64,
                            device="cuda")
        if tuple(F.shape) != (d, d):
            raise DimensionMismatch(f"head {i + 1} must be ({d}, {d}), got {tuple(F.shape)}")
        hs.append(hs[-1] @ F + hs[-1])
    return torch.stack([E @ x for x in hs])


def _validate(req: ForwardRequest, max_positions: int) -> int:
    """model.py:123-143."""
    if not req.tokens:
        raise ValueError("forward request must contain at least one token")
    if len(req.tokens) != len(req.positions):
        raise ValueError("tokens and positions must have equal length")
    for p in req.positions:
        if p >= max_positions:
            raise PositionOverflow(f"position {p} >= max_positions {max_positions}")
    ctx = len(req.cache)
    if req.attention_mask is not None:
        m = np.asarray(req.attention_mask, dtype=bool)
        want = (len(req.tokens), ctx + len(req.tokens))
        if m.shape != want:
            raise MaskShapeMismatch(f"mask shape {m.shape}, expected {want}")
        if not m[:, :ctx].all():
            raise ValueError("cache entries must be visible to every row")
        if not all(m[r, ctx + r] for r in range(len(req.tokens))):
            raise ValueError("every row must attend to itself")
    return ctx


def _splits(y: torch.Tensor) -> tuple[int, int]:
    """(slices, elements between slices) of a dense() output: [S, T, N] split-K
    slices from sd_gemm or a plain [T, N] product."""
    if y.dim() == 3:
        return y.shape[0], y.shape[1] * y.shape[2]
    return 1, 0


def mask_bits_from_bool(block: np.ndarray) -> np.ndarray:
    """(T, T) bool over request rows -> int32 [T][MASK_WORDS] bit rows
    (only j <= r is honoured, like _row_ancestors, model.py:146-147)."""
    T = block.shape[0]
    bits = np.zeros((T, L.MASK_WORDS), dtype=np.uint32)
    for r in range(T):
        for j in np.nonzero(block[r, : r + 1])[0]:
            bits[r, j >> 5] |= np.uint32(1 << (j & 31))
    return bits.view(np.int32)


class TinyTransformer:
    """Device model. `params` may be a dict of numpy/torch arrays in the
    reference layout; otherwise weights come from the reference's seeded
    streams (init="reference", exact) or torch's device RNG with the same
    scales (init="device", fast for multi-GB configs)."""

    def __init__(self, config: ModelConfig, params: dict | None = None, *, dtype: torch.dtype = torch.bfloat16,
                 device: str | torch.device = "cuda", init: str = "reference", shard: tuple[int, int] = (0, 1),
                 group=None):
        L.require_cuda()
        L.load()
        self.config = c = config
        self.dtype, self.device = dtype, torch.device(device)
        self.rank, self.world = shard
        self.group = group
        if c.num_kv_heads % self.world:
            raise ValueError(f"{c.num_kv_heads} kv heads cannot be sharded over {self.world} ranks")
        self.Hk = c.num_kv_heads // self.world
        self.H = self.Hk * c.group_size
        self.dh = c.head_dim
        self.q_scale = float(1.0 / math.sqrt(c.head_dim))
        self._load_weights(params, init)
        # RoPE tables from fp64 angles (model.py:161, 276-277), fp32 storage
        half = c.head_dim // 2
        inv = 10000.0 ** (-np.arange(0, c.head_dim, 2) / c.head_dim)
        ang = np.arange(c.max_positions, dtype=np.float64)[:, None] * inv[None, :]
        self.rope_cos = torch.as_tensor(np.cos(ang).astype(np.float32), device=self.device).reshape(-1, half)
        self.rope_sin = torch.as_tensor(np.sin(ang).astype(np.float32), device=self.device).reshape(-1, half)
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self.use_tc = True  # tcgen05 verification attention when the cache supports it

    # ------------------------------------------------------------ weights --
    def _load_weights(self, params, init):
        c, dev, dt = self.config, self.device, self.dtype
        specs = param_specs(c)
        gen = None
        if params is None and init == "device":
            gen = torch.Generator(device=dev)
            gen.manual_seed(c.init_seed)

        def get(idx, name, shape, scale):
            if params is not None:
                a = params[name]
                return torch.as_tensor(a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a),
                                       dtype=torch.float64).to(dev)
            if init == "device":
                if scale == 0.0:
                    return torch.ones(shape, dtype=torch.float32, device=dev)
                t = torch.empty(shape, dtype=torch.float32, device=dev)
                t.normal_(0.0, scale, generator=gen)
                return t
            return torch.as_tensor(reference_tensor(c, idx, shape, scale), dtype=torch.float64).to(dev)

        from .parallel import shard_heads
        (q0, q1), (k0, k1) = shard_heads(c.num_heads, c.num_kv_heads, c.head_dim, self.rank, self.world)
        self.layers = []
        cur: dict = {}
        for idx, (name, shape, scale) in enumerate(specs):
            t = get(idx, name, shape, scale)
            if name == "embed":
                self.embed = t.to(dt).contiguous()
            elif name == "ln_f":
                self.ln_f = t.float().contiguous()
            elif name.startswith("head"):
                self.heads = getattr(self, "heads", [])
                self.heads.append(t.to(dt).contiguous())
            else:
                key = name.split(".")[1]
                cur[key] = t
                if key == "w2":
                    wqkv = torch.cat([cur["wq"][:, q0:q1], cur["wk"][:, k0:k1], cur["wv"][:, k0:k1]], dim=1)
                    self.layers.append({
                        "ln1": cur["ln1"].float().contiguous(), "wqkv": wqkv.to(dt).contiguous(),
                        "wo": cur["wo"].to(dt).contiguous(), "ln2": cur["ln2"].float().contiguous(),
                        "w1": cur["w1"].to(dt).contiguous(), "w2": cur["w2"].to(dt).contiguous(),
                    })
                    cur = {}
            del t
        if not hasattr(self, "heads"):
            self.heads = []
        self._gemm_ws = None
        keys = os.environ.get("SD_GEMM_KEYS")  # tuning switch: comma list of projections for sd_gemm
        if keys is not None:
            self.use_gemm = bool(keys)
            self.gemm_keys = tuple(k for k in keys.split(",") if k)
        if dt == torch.bfloat16 and self.use_gemm:
            self._make_gemm_maps()
        self._gemv_ws = None
        if dt == torch.bfloat16:
            need = 256
            for ly in self.layers:
                for key in ("wqkv", "wo", "w1", "w2"):
                    need = max(need, L.load().sd_gemv_workspace_bytes(*ly[key].shape))
            for f in self.heads:
                need = max(need, L.load().sd_gemv_workspace_bytes(*f.shape))
            self._gemv_ws = torch.zeros(need, dtype=torch.uint8, device=dev)
        torch.cuda.empty_cache()

    # Weight-streaming tcgen05 GEMM (sd_gemm) for the decode rows. Off by
    # default: routed per projection (SD_GEMM_KEYS=wqkv,wo,...) the cfg3 step
    # is slower than with cuBLAS for every subset (8.78 ms with none, 8.95 with
    # wqkv, 9.24 with wqkv+wo, 9.88 with all; profiles/r01_gemm_keys_sweep.log),
    # so the product path keeps cuBLAS for the verify forward's dense layers.
    use_gemm = False
    gemm_keys = ("wqkv", "wo", "w1", "w2")

    def _make_gemm_maps(self):
        """N-tiled copies [N/128][K][128] of the layer weights for sd_gemm (the
        row-major originals stay for cuBLAS prefill)."""
        import ctypes
        need = 0
        for ly in self.layers:
            for key in self.gemm_keys:
                K, N = ly[key].shape
                if K % 64 or N % 128:
                    continue
                wt = torch.empty((N // 128, 2, K, 64), dtype=self.dtype, device=self.device)
                L.call("sd_tile_weight", L.ptr(ly[key]), K, N, L.ptr(wt), L.stream())
                tm = ctypes.create_string_buffer(128)
                L.call("sd_make_weight_tmap", L.ptr(wt), K, N, tm)
                ly["wt_" + key], ly["tm_" + key] = wt, tm
                need = max(need, L.load().sd_gemm_workspace_bytes(16, N, K))
        self._gemm_ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device)

    # single-row (draft) projections stream their weights with sd_gemv
    use_gemv = True

    def gemv(self, x: torch.Tensor, w: torch.Tensor, silu: bool = False) -> torch.Tensor:
        """[1, K] bf16 @ w [K, N] -> [1, N] fp32 (bf16 silu(.) with silu=True)."""
        K, N = w.shape
        y = torch.empty((1, N), dtype=self.dtype if silu else torch.float32, device=self.device)
        L.call("sd_gemv", L.ptr(x), K, L.ptr(w), N, L.GEMM_EPI_SILU_BF16 if silu else L.GEMM_EPI_F32, L.ptr(y),
               L.ptr(self._gemv_ws), self._gemv_ws.numel(), L.stream())
        return y

    def _gemv_ok(self, x: torch.Tensor, w: torch.Tensor) -> bool:
        return (self.use_gemv and self._gemv_ws is not None and x.shape[0] == 1 and x.dtype == torch.bfloat16
                and x.is_contiguous() and w.shape[1] % 8 == 0)

    def dense_norm(self, x: torch.Tensor, ly: dict, key: str, h: torch.Tensor, gain: torch.Tensor,
                   out_dtype=None) -> torch.Tensor:
        """norm(h, x @ ly[key], gain): h += x @ w, returns rmsnorm(h) * gain. One
        launch (sd_gemv_addnorm) for the single draft row, else dense() + norm()."""
        dt = out_dtype or self.dtype
        if self.fuse_norm and h.shape[0] == 1 and self._gemv_ok(x, ly[key]):
            K, N = ly[key].shape
            out = torch.empty((1, N), dtype=dt, device=self.device)
            L.call("sd_gemv_addnorm", L.ptr(x), K, L.ptr(ly[key]), N, L.ptr(h), L.ptr(gain), 1e-6, L.ptr(out),
                   L.dcode(dt), L.ptr(self._gemv_ws), self._gemv_ws.numel(), L.stream())
            return out
        return self.norm(h, self.dense(x, ly, key), gain, out_dtype=out_dtype)

    # the single-row projection + residual add + RMSNorm as one launch
    # (sd_gemv_addnorm). Off: the serial row tail inside the projection costs more
    # (+4.4 us per launch) than the separate RMSNorm launch it removes, which
    # overlaps the next projection's weight prefetch (cfg3 step 8.69 vs 8.47 ms).
    fuse_norm = False

    # few-row weight streaming (sd_gemm_rows, tcgen05 swap-AB) for the verification
    # forward's projections whose consumers take split-K slices (RoPE staging,
    # residual add + RMSNorm); rows_hint: the tree record's live row count (device
    # int), set by the engine around the verify forward (padded graph rows are
    # skipped). Off by default: faster than cuBLAS per projection when timed alone
    # (qkv 10.5 vs 12.1 us, wo 8.5 vs 9.3 us), but the cfg3 step is 0.16-0.3 ms
    # slower with it (the consumers re-read 6-9 fp32 slices per row; per-launch
    # ramp), profiles/r02_gemm_rows_experiment.txt. SD_ROWS_KEYS=wqkv,wo turns it on.
    rows_keys = tuple(k for k in os.environ.get("SD_ROWS_KEYS", "").split(",") if k)
    rows_hint: torch.Tensor | None = None

    def _rows_ok(self, x: torch.Tensor, w: torch.Tensor, key: str) -> bool:
        K, N = w.shape
        return (key in self.rows_keys and self.dtype == torch.bfloat16 and x.dtype == torch.bfloat16
                and x.is_contiguous() and 1 < x.shape[0] <= 112 and K % 32 == 0 and N % 256 == 0)

    def gemm_rows(self, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        """x [T, K] bf16 @ w [K, N] -> [S, T, N] fp32 split-K slices (sd_gemm_rows)."""
        if L.DEBUG_SKIP and f"mm:{w.shape[1]}" in L.DEBUG_SKIP:  # profiling only
            return torch.empty((1, x.shape[0], w.shape[1]), dtype=torch.float32, device=x.device)
        K, N = w.shape
        T = x.shape[0]
        y = torch.empty((L.load().sd_gemm_rows_splits(K, N), T, N), dtype=torch.float32, device=self.device)
        L.call("sd_gemm_rows", L.ptr(x), T, K, L.ptr(w), N, L.ptr(self.rows_hint), L.ptr(y), L.stream())
        return y

    def dense(self, x: torch.Tensor, ly: dict, key: str, silu: bool = False) -> torch.Tensor:
        """x @ ly[key] -> fp32 [T, N], or [S, T, N] split-K slices whose in-order
        sum is the product (consumed by norm() / rope_stage()); silu=True gives
        bf16 silu(x @ w) (the MLP up-projection)."""
        if self._gemv_ok(x, ly[key]):
            return self.gemv(x, ly[key], silu)
        if not silu and self._rows_ok(x, ly[key], key):
            return self.gemm_rows(x, ly[key])
        tm = ly.get("tm_" + key)
        T = x.shape[0]
        if tm is None or T > 128 or not self.use_gemm or not x.is_contiguous():
            y = self.mm(x, ly[key])
            return self.silu(y) if silu else y
        K, N = ly[key].shape
        epi = L.GEMM_EPI_SILU_BF16 if silu else L.GEMM_EPI_F32
        S = L.load().sd_gemm_splits(T, N, K, epi)
        y = torch.empty((T, N) if silu else (S, T, N), dtype=self.dtype if silu else torch.float32,
                        device=self.device)
        L.call("sd_gemm", L.ptr(x), T, K, tm, N, epi, L.ptr(y), N, L.ptr(self._gemm_ws), self._gemm_ws.numel(),
               L.stream())
        return y

    def parameters_host(self) -> dict:
        """Weights back in the reference layout (fp64 numpy; shard-local)."""
        c = self.config
        out = {"embed": self.embed.double().cpu().numpy(), "ln_f": self.ln_f.double().cpu().numpy()}
        qd, kd = self.H * self.dh, self.Hk * self.dh
        for i, ly in enumerate(self.layers):
            w = ly["wqkv"].double().cpu().numpy()
            out[f"l{i}.wq"], out[f"l{i}.wk"], out[f"l{i}.wv"] = w[:, :qd], w[:, qd:qd + kd], w[:, qd + kd:]
            for k in ("ln1", "wo", "ln2", "w1", "w2"):
                out[f"l{i}.{k}"] = ly[k].double().cpu().numpy()
        for i, f in enumerate(self.heads):
            out[f"head{i + 1}"] = f.double().cpu().numpy()
        return out

    def weight_bytes(self) -> int:
        n = self.embed.numel() * self.embed.element_size() + self.ln_f.numel() * 4
        for ly in self.layers:
            n += sum(t.numel() * t.element_size() for t in ly.values())
        n += sum(f.numel() * f.element_size() for f in self.heads)
        return n

    # -------------------------------------------------------------- caches --
    def new_cache(self, capacity: int | None = None) -> FullCache:
        cap = capacity or min(self.config.max_positions + L.TREE_MAX_ROWS, 1 << 16)
        return FullCache(self.config.num_layers, self.Hk, self.dh, cap, self.dtype, self.device)

    def new_partial(self, sink: int, budget: int) -> PartialCache:
        return PartialCache(sink, budget, self.config.num_layers, self.Hk, self.dh, self.dtype, self.device)

    # ---------------------------------------------------------- primitives --
    def mm(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        if L.DEBUG_SKIP and f"mm:{b.shape[1]}" in L.DEBUG_SKIP:  # profiling only (see _lib.DEBUG_SKIP)
            return torch.empty((a.shape[0], b.shape[1]), dtype=torch.float32, device=a.device)
        if self.dtype == torch.bfloat16:
            return torch.mm(a, b, out_dtype=torch.float32)
        return torch.mm(a, b)

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws.numel() < nbytes:  # zeroed: sd_attention keeps arrival counters in its head
            self._ws = torch.zeros(int(nbytes * 1.25) + 1024, dtype=torch.uint8, device=self.device)
        return self._ws

    def _gather_heads(self, o: torch.Tensor) -> torch.Tensor:
        """[T, H_local*dh] -> [T, H*dh] (NCCL all-gather over kv-head shards)."""
        if self.world == 1:
            return o
        from .parallel import all_gather_heads
        return all_gather_heads(o, self.world, self.group)

    def attention(self, q_rot, T, src_kind, k_cache, v_cache, head_stride, ctx, ranks, k_tree, v_tree,
                  tree_head_stride, mask_bits, rows_dev, out, tmaps=None, layer=0, ctx_dev=None, ws=None):
        """sd_attention; with `tmaps` (FullCache.tmaps) and bf16/dh=128 the cache
        chunks run on the tcgen05 kernel of `layer` (PartialCache.tmaps: the
        tensor-core draft kernel). With `ctx_dev` the live
        context is read on device and `ctx` is its upper bound (graph replay).
        `ws`: caller-owned workspace (a Session's, sized once and captured in its
        graph); default the model's scratch, which may be reallocated."""
        nbytes = L.load().sd_attention_workspace_bytes(T, self.H, self.dh, ctx)
        if ws is None:
            ws = self.workspace(nbytes)
        elif ws.numel() < nbytes:
            raise ValueError(f"attention workspace {ws.numel()} B < {nbytes} B")
        kd = L.dcode(self.dtype)
        tk, tv = tmaps if (tmaps is not None and self.use_tc) else (None, None)
        L.call("sd_attention", L.ptr(q_rot), kd, T, self.H, self.Hk, self.dh, src_kind, L.ptr(k_cache),
               L.ptr(v_cache), kd, head_stride, ctx, L.ptr(ranks), L.ptr(self.rope_cos), L.ptr(self.rope_sin),
               L.ptr(k_tree), L.ptr(v_tree), tree_head_stride, L.ptr(mask_bits),
               L.MASK_WORDS if mask_bits is not None else 0, L.ptr(rows_dev), L.ptr(ctx_dev), tk, tv, layer,
               self.config.num_kv_heads, L.ptr(out), kd, L.ptr(ws), ws.numel(), L.stream())

    def rope_stage(self, qkv, T, positions_dev, q_rot, q_pre, k_raw, k_rot, v, head_stride, row_offset,
                   rows_dev=None):
        kd = L.dcode(self.dtype)
        S, sstride = _splits(qkv)
        L.call("sd_rope_stage", L.ptr(qkv), T, self.H, self.Hk, self.dh, L.ptr(positions_dev),
               L.ptr(self.rope_cos), L.ptr(self.rope_sin), self.q_scale, L.ptr(q_rot), kd, L.ptr(q_pre),
               L.ptr(k_raw), L.ptr(k_rot), L.ptr(v), kd, head_stride, row_offset, L.ptr(rows_dev), S, sstride,
               L.stream())

    def norm(self, h, delta, gain, out_dtype=None):
        T, d = h.shape
        dt = out_dtype or self.dtype
        x = torch.empty((T, d), dtype=dt, device=self.device)
        S, sstride = _splits(delta) if delta is not None else (1, 0)
        L.call("sd_add_rmsnorm", L.ptr(h), L.ptr(delta), T, d, L.ptr(gain), 1e-6, L.ptr(x), L.dcode(dt), S, sstride,
               L.stream())
        return x

    def embed_rows(self, tokens_dev, T):
        h = torch.empty((T, self.config.hidden_dim), dtype=torch.float32, device=self.device)
        L.call("sd_embed", L.ptr(tokens_dev), T, L.ptr(self.embed), L.dcode(self.dtype), self.config.hidden_dim,
               L.ptr(h), L.stream())
        return h

    silu_rows = os.environ.get("SD_SILU_ROWS", "1") != "0"  # A/B switch (tools only)

    def silu(self, a):
        out = torch.empty(a.shape, dtype=self.dtype, device=self.device)
        if self.silu_rows and self.rows_hint is not None and a.dim() == 2 and a.shape[1] % 4 == 0:  # skip padding
            L.call("sd_silu_rows", L.ptr(a), L.ptr(out), L.dcode(self.dtype), a.shape[0], a.shape[1],
                   L.ptr(self.rows_hint), L.stream())
            return out
        L.call("sd_silu", L.ptr(a), L.ptr(out), L.dcode(self.dtype), a.numel(), L.stream())
        return out

    # -------------------------------------------------------- layer stack --
    # single-row (draft) forward with each residual add + RMSNorm folded into the
    # next projection's input load (sd_gemv_norm): 2 norm launches per layer fewer
    fuse_row_norms = os.environ.get("SD_FUSE_ROW_NORMS", "1") != "0"  # A/B switch (tools only)

    def _row_fused_ok(self) -> bool:
        return (self.fuse_row_norms and self.use_gemv and self._gemv_ws is not None and self.dtype == torch.bfloat16
                and self.config.hidden_dim % 8 == 0)

    def gemv_norm(self, h_in, delta, gain, h_out, w, silu: bool = False) -> torch.Tensor:
        """h_out = h_in + delta; y = bf16(rmsnorm(h_out) * gain) @ w in one launch."""
        K, N = w.shape
        y = torch.empty((1, N), dtype=self.dtype if silu else torch.float32, device=self.device)
        L.call("sd_gemv_norm", L.ptr(h_in), L.ptr(delta), L.ptr(gain), 1e-6, L.ptr(h_out), K, L.ptr(w), N,
               L.GEMM_EPI_SILU_BF16 if silu else L.GEMM_EPI_F32, L.ptr(y), L.ptr(self._gemv_ws),
               self._gemv_ws.numel(), L.stream())
        return y

    # the draft row's RoPE + staging folded into its QKV projection (sd_gemv_rope):
    # one launch per layer fewer. A/B switch: tools only.
    fuse_draft_rope = os.environ.get("SD_FUSE_DRAFT_ROPE", "1") != "0"

    def gemv_rope(self, x, pending, w, rope, h_out=None) -> None:
        """One-row QKV projection whose epilogue rotates Q/K at the device position
        rope[0] and writes q_rot (scaled) / k / v (rope = (pos, q_rot, k, v))."""
        K, N = w.shape
        pos, q_rot, k, v = rope
        if pending is None:
            args = (L.ptr(x), None, None, None, 1e-6, None)
        else:
            args = (None, L.ptr(pending[0]), L.ptr(pending[1]), L.ptr(pending[2]), 1e-6, L.ptr(h_out))
        L.call("sd_gemv_rope", *args, K, L.ptr(w), N, L.ptr(pos), L.ptr(self.rope_cos), L.ptr(self.rope_sin),
               self.q_scale, self.H, self.Hk, self.dh, L.ptr(q_rot), L.ptr(k), L.ptr(v), L.ptr(self._gemv_ws),
               self._gemv_ws.numel(), L.stream())

    def _run_layers_row(self, tokens_dev, attend, q_pre=None, rope=None):
        """run_layers for one row (the draft forward) with the norms fused into
        the weight streams; the residual stream ping-pongs between two rows.
        With `rope` the QKV projections also rotate and stage the row, and
        attend() receives qkv = None."""
        h = self.embed_rows(tokens_dev, 1)
        other = torch.empty_like(h)
        x = self.norm(h, None, self.layers[0]["ln1"])
        pending = None  # (h, delta, gain) of the norm that feeds the next projection
        nl = len(self.layers)
        rope = rope if (rope is not None and self.fuse_draft_rope) else None
        for l, ly in enumerate(self.layers):
            if rope is not None:
                qkv = None
                self.gemv_rope(x if pending is None else None, pending, ly["wqkv"], rope, h_out=other)
                if pending is not None:
                    h, other = other, h
            elif pending is None:
                qkv = self.gemv(x, ly["wqkv"])
            else:
                qkv = self.gemv_norm(pending[0], pending[1], pending[2], other, ly["wqkv"])
                h, other = other, h
            o = self._gather_heads(attend(l, qkv, None if q_pre is None else q_pre[l]))
            d1 = self.gemv(o, ly["wo"])
            a = self.gemv_norm(h, d1, ly["ln2"], other, ly["w1"], silu=True)
            h, other = other, h
            d2 = self.gemv(a, ly["w2"])
            if l + 1 < nl:
                pending = (h, d2, self.layers[l + 1]["ln1"])
            else:
                return self.norm(h, d2, self.ln_f, out_dtype=torch.float32)  # h0 (fp32)

    def run_layers(self, tokens_dev, T, attend, q_pre=None, rope=None):
        """Embedding + L layers + final norm. attend(l, qkv, q_pre_l) -> [T, H_local*dh].
        Returns h0 = rmsnorm(h, ln_f) in fp32 [T, d]. rope (one row only): see
        _run_layers_row."""
        if T == 1 and self._row_fused_ok():
            return self._run_layers_row(tokens_dev, attend, q_pre, rope)
        h = self.embed_rows(tokens_dev, T)
        x = self.norm(h, None, self.layers[0]["ln1"])
        nl = len(self.layers)
        for l, ly in enumerate(self.layers):
            qkv = self.dense(x, ly, "wqkv")
            o = attend(l, qkv, None if q_pre is None else q_pre[l])
            o = self._gather_heads(o)
            x = self.dense_norm(o, ly, "wo", h, ly["ln2"])
            a = self.dense(x, ly, "w1", silu=True)
            last = l + 1 == nl
            x = self.dense_norm(a, ly, "w2", h, self.ln_f if last else self.layers[l + 1]["ln1"],
                                out_dtype=torch.float32 if last else None)
        return x  # fp32 h0

    def head_logits(self, h0: torch.Tensor, heads: int) -> torch.Tensor:
        """Chained draft heads on the LAST row of h0 ([1, d] fp32) -> [heads, V] fp32."""
        hs = [h0]
        for i in range(heads - 1):
            xb = hs[-1].to(self.dtype)
            d = self.gemv(xb, self.heads[i]) if self._gemv_ok(xb, self.heads[i]) else self.mm(xb, self.heads[i])
            hs.append(hs[-1] + d)
        stack = torch.cat(hs, dim=0).to(self.dtype)
        return self.mm(stack, self.embed.t())

    def lm_logits(self, h0: torch.Tensor) -> torch.Tensor:
        return self.mm(h0.to(self.dtype), self.embed.t())

    # verification LM head fused with the penalty + softmax statistics of the
    # sampler (sd_lmhead_sample_stats). A/B switch: tools only.
    fuse_lm_head = os.environ.get("SD_FUSE_LM_HEAD", "1") != "0"

    def lmhead_fused_ok(self, T: int) -> bool:
        return (self.fuse_lm_head and self.dtype == torch.bfloat16 and self.device.type == "cuda" and 0 < T <= 128
                and self.config.hidden_dim % 64 == 0 and self.embed.is_contiguous())

    def lm_head_sample_stats(self, h0: torch.Tensor, args, logits_out: torch.Tensor, stats_out: torch.Tensor,
                             x_buf: torch.Tensor | None = None) -> None:
        """logits_out [T, V] = penalised scaled logits, stats_out [T, tiles, 2]
        = per-128-token (max, sum-exp), for the penalty fields of `args`
        (an L.SampleArgs) — one tcgen05 launch streaming the tied embedding."""
        import ctypes
        if getattr(self, "_lm_tmap", None) is None:
            V, d = self.config.vocab_size, self.config.hidden_dim
            # box-contiguous copy of the tied embedding (+1.05 GB at cfg3), made once
            self._lm_tiled = torch.empty(L.load().sd_lmhead_tiled_bytes(V, d), dtype=torch.uint8, device=self.device)
            L.call("sd_tile_lmhead", L.ptr(self.embed), V, d, L.ptr(self._lm_tiled), L.stream())
            self._lm_tmap = ctypes.create_string_buffer(128)
            L.call("sd_make_lmhead_tmap", L.ptr(self._lm_tiled), V, d, self._lm_tmap)
        T = h0.shape[0]
        x = x_buf if x_buf is not None else torch.empty((T, h0.shape[1]), dtype=self.dtype, device=self.device)
        x.copy_(h0)
        L.call("sd_lmhead_sample_stats", L.ptr(x), T, self.config.hidden_dim, self._lm_tmap, self.config.vocab_size,
               args, L.ptr(logits_out), L.ptr(stats_out), L.stream())

    # ------------------------------------------------------ generic API ----
    def forward(self, req: ForwardRequest) -> ForwardResult:
        """Reference forward contract (model.py:251-313) on device."""
        c = self.config
        ctx = _validate(req, c.max_positions)
        T = len(req.tokens)
        cache = req.cache
        dev = self.device
        toks = torch.tensor([int(t) for t in req.tokens], dtype=torch.int32, device=dev)
        pos = torch.tensor([int(p) for p in req.positions], dtype=torch.int32, device=dev)
        queries = torch.empty((c.num_layers, T, self.H, self.dh), dtype=torch.float32, device=dev)
        q_rot = torch.empty((T, self.H, self.dh), dtype=self.dtype, device=dev)
        if isinstance(cache, DraftView):
            attend = self._draft_attend_fn(cache.partial, T, pos, q_rot, causal_mask=req.attention_mask)
        else:
            cache.reserve(T)
            attend = self._full_attend_fn(cache, ctx, T, pos, q_rot, req.attention_mask)
        h0 = self.run_layers(toks, T, attend, q_pre=queries)
        heads = c.gamma + 1 if req.heads_needed is None else min(req.heads_needed, c.gamma + 1)
        bundles = torch.full((T, c.gamma + 1, c.vocab_size), -math.inf, dtype=torch.float32, device=dev)
        if heads == 1:
            bundles[:, 0] = self.lm_logits(h0)
        else:
            for r in range(T):
                bundles[r, :heads] = self.head_logits(h0[r:r + 1], heads)
        if not isinstance(cache, DraftView):
            cache.commit_rows(req.positions)
        return ForwardResult(bundles=bundles, queries=queries.permute(1, 0, 2, 3))

    def _full_attend_fn(self, cache: FullCache, ctx, T, pos, q_rot, mask):
        out = torch.empty((T, self.H * self.dh), dtype=self.dtype, device=self.device)
        if mask is not None:
            if T > L.TREE_MAX_ROWS:
                raise ValueError(f"masked forward supports at most {L.TREE_MAX_ROWS} rows")
            bits = torch.as_tensor(mask_bits_from_bool(np.asarray(mask, dtype=bool)[:, ctx:]), device=self.device)
        else:
            bits = None

        def attend(l, qkv, q_pre):
            self.rope_stage(qkv, T, pos, q_rot, q_pre, cache.k_raw[l, :, ctx:], cache.k_rot[l, :, ctx:],
                            cache.v[l, :, ctx:], cache.head_stride, 0)
            if bits is not None:
                self.attention(q_rot, T, 0, cache.k_rot[l], cache.v[l], cache.head_stride, ctx, None,
                               cache.k_rot[l, :, ctx:], cache.v[l, :, ctx:], cache.head_stride, bits, None, out,
                               cache.tmaps, l)
            else:  # causal in blocks of <= 128 rows (model.py:301-305)
                for b0 in range(0, T, 128):
                    tb = min(128, T - b0)
                    self.attention(q_rot[b0:], tb, 0, cache.k_rot[l], cache.v[l], cache.head_stride, ctx + b0,
                                   None, cache.k_rot[l, :, ctx + b0:], cache.v[l, :, ctx + b0:], cache.head_stride,
                                   None, None, out[b0:], cache.tmaps, l)
            return out
        return attend

    def _draft_attend_fn(self, partial: PartialCache, T, pos, q_rot, causal_mask=None):
        out = torch.empty((T, self.H * self.dh), dtype=self.dtype, device=self.device)
        kt = torch.empty((self.Hk, T, self.dh), dtype=self.dtype, device=self.device)
        vt = torch.empty_like(kt)
        if T > L.TREE_MAX_ROWS:
            raise ValueError("draft forward rows exceed device limit")

        def attend(l, qkv, q_pre):
            self.rope_stage(qkv, T, pos, q_rot, q_pre, None, kt, vt, T * self.dh, 0)
            self.attention(q_rot, T, 1, partial.pk[l], partial.pv[l], partial.head_stride, partial.hi,
                           partial.prank[l], kt, vt, T * self.dh, None, None, out,
                           partial.tmaps if T == 1 else None, l)
            return out
        return attend
