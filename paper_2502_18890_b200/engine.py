"""Generation engine on B200 (API mirror of swiftdec/engine.py).

Session.step() is Algorithm 1 (engine.py:185-302) with every stage on device:

  draft forward over the partial cache (sd_attention src=1, rank RoPE on load)
  -> chained draft heads -> sd_draft_topw (penalised per-head top-w)
  -> sd_draft_tree (n-gram retrieval + candidate tree, one CTA)
  -> verification forward, padded to the tree's max rows with the live row
     count read on device (sd_rope_stage / sd_attention rows_dev)
  -> sd_sample_rows (per-row window splice, penalty, truncation, draw)
  -> sd_accept_commit (paths, uniform pick, window / history / n-gram commit)
  -> sd_reconcile (accepted rows + last_queries)
  -> sd_partial_step (admit + evict, slot bookkeeping on device)
  -> one 128-byte device->host copy of the step result.

The only host round trip per step is that result copy (the step record the
API returns); the refresh decision is integer arithmetic on host counters
that mirror the device state exactly, and a refresh is one fused launch
(sd_partial_refresh) before the step's graph.

Graph mode (default): every launch from the draft forward to the result copy
takes only step-invariant arguments — the committed length lives on device
(state[SD_ST_BASE], advanced by sd_accept_commit; the verify rows' cache
offset and the attention context are read from the tree record), the draft
attention scans the whole slot range (holes are masked by rank < 0) — so the
step is captured once as a CUDA graph and replayed; per step the host issues
one graph launch (plus a refresh launch every B - S tokens).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .kvcache import FullCache, PartialCache, needs_refresh
from .metrics import IterationRecord, RunMetrics, collect_metrics
from .model import PositionOverflow, TinyTransformer
from .ngram import NGramTable
from .rng import derive_seed
from .sampling import PenaltyWindow, SamplerConfig
from .tree import TreeConfig


class ConfigError(ValueError):
    """Engine configuration violates an invariant."""


class PromptTooShort(ConfigError):
    """Prompt shorter than the cache sink."""


class SessionExhausted(RuntimeError):
    """step() called after the target length was reached."""


@dataclass(frozen=True)
class EngineConfig:
    target_length: int
    sink_size: int = 32
    budget: int = 1024
    tree: TreeConfig = field(default_factory=TreeConfig)
    k: int = 20
    sampler: SamplerConfig = field(default_factory=SamplerConfig)
    seed: int = 0
    bonus: bool = True

    def validate(self, gamma: int) -> None:
        """engine.py:70-85."""
        if self.target_length < 1:
            raise ConfigError("target_length must be >= 1")
        if self.budget <= self.sink_size:
            raise ConfigError("budget must exceed sink_size")
        if self.budget - self.sink_size < gamma + 2:
            raise ConfigError("budget - sink_size must be at least gamma + 2 to fit one iteration's acceptance")
        if self.tree.depth != gamma + 1:
            raise ConfigError(f"tree depth {self.tree.depth} must equal gamma + 1 = {gamma + 1}")
        if self.k < 0:
            raise ConfigError("k must be >= 0")
        if self.k > 64:
            raise ConfigError("k above the device n-gram limit of 64")
        if self.tree.depth > L.TREE_MAX_DEPTH:
            raise ConfigError(f"tree depth above {L.TREE_MAX_DEPTH}")
        if self.tree.max_rows(self.k) > L.TREE_MAX_ROWS or self.tree.head_leaves + self.k > L.TREE_MAX_PATHS:
            raise ConfigError("tree too large for the device record")
        if self.budget - self.sink_size > 8192:
            raise ConfigError("partial-cache body above the device top-K limit of 8192")


def _trunc_fields(args: L.SampleArgs, smp: SamplerConfig) -> None:
    args.temperature, args.theta, args.ctrl_style = smp.temperature, smp.theta, int(smp.ctrl_style)
    args.trunc_kind = smp.truncation.code
    args.trunc_value = smp.truncation.value
    args.eta_alpha = smp.truncation.eta_alpha if smp.truncation.eta_alpha is not None else -1.0
    args.seed = smp.seed & ((1 << 64) - 1)


class Session:
    """One speculative generation run; owns its device caches and tables."""

    def __init__(self, model: TinyTransformer, prompt: list[int], config: EngineConfig,
                 capacity: int | None = None, prefill: bool = True, graph: bool = True):
        c = model.config
        gamma = c.gamma
        config.validate(gamma)
        if len(prompt) <= config.sink_size:
            raise PromptTooShort(f"prompt length {len(prompt)} must exceed the sink size {config.sink_size} "
                                 "(sink entries plus the decoding root)")
        self.model, self.config = model, config
        self.gamma, self.depth = gamma, gamma + 1
        self.tokens = [int(t) for t in prompt]
        self.prompt_len = len(prompt)
        self.emitted: list[int] = []
        self.records: list[IterationRecord] = []
        self.select_seed = derive_seed(config.seed, "branch-select")
        self.wall_times = {"prefill": 0.0, "draft": 0.0, "verify": 0.0}
        self.forward_counts = {"prefill": 0, "draft": 0, "verify": 0}
        dev = model.device
        self.dev = dev
        V = c.vocab_size
        self.Tmax = config.tree.max_rows(config.k)
        # ---- device state ----
        self.state = torch.zeros(16, dtype=torch.int64, device=dev)
        self.result = torch.zeros(32, dtype=torch.int32, device=dev)
        self.result_host = torch.zeros(32, dtype=torch.int32, pin_memory=True)
        self.tree_rec = torch.zeros(L.tree_layout()["TOTAL"], dtype=torch.int32, device=dev)
        self.per_head = torch.zeros(sum(config.tree.widths), dtype=torch.int32, device=dev)
        self.grams = torch.zeros(64 * self.depth, dtype=torch.int32, device=dev)
        self.y = torch.zeros(L.TREE_MAX_ROWS, dtype=torch.int32, device=dev)
        self.history = torch.zeros(config.target_length + 2 * self.depth + 8, dtype=torch.int32, device=dev)
        self.window = PenaltyWindow(config.sampler.window, V, state=self.state, device=dev)
        ng_cap = 1
        while ng_cap < 2 * (config.target_length + 2 * self.depth) + 16:
            ng_cap <<= 1
        self.ngrams = NGramTable(n=self.depth, k_max=max(64, config.k), capacity=ng_cap, vocab_size=V, device=dev)
        cap = capacity or (len(prompt) + config.target_length + self.depth + self.Tmax + 8)
        self.full: FullCache = model.new_cache(cap)
        self.q_pre = torch.zeros((c.num_layers, self.Tmax, model.H, model.dh), dtype=torch.float32, device=dev)
        self.q_sum = torch.zeros((c.num_layers, model.H, model.dh), dtype=torch.float32, device=dev)
        self.q_rot_v = torch.zeros((self.Tmax, model.H, model.dh), dtype=model.dtype, device=dev)
        self.q_rot_d = torch.zeros((1, model.H, model.dh), dtype=model.dtype, device=dev)
        self.kt = torch.zeros((model.Hk, 1, model.dh), dtype=model.dtype, device=dev)
        self.vt = torch.zeros_like(self.kt)
        self.attn_out_v = torch.zeros((self.Tmax, model.H * model.dh), dtype=model.dtype, device=dev)
        self.attn_out_d = torch.zeros((1, model.H * model.dh), dtype=model.dtype, device=dev)
        self.partial: PartialCache | None = None
        # Session-owned attention workspace (split partials + the draft kernel's
        # arrival counters, zeroed once): sized for the largest verify context and
        # the draft slot range up front, so the captured graph never sees it move
        # and sessions sharing a model never share scratch.
        slot_cap = config.budget + L.TREE_MAX_DEPTH
        lib = L.load()
        self.attn_ws = torch.zeros(max(lib.sd_attention_workspace_bytes(self.Tmax, model.H, model.dh, cap),
                                       lib.sd_attention_workspace_bytes(1, model.H, model.dh, max(slot_cap, cap))),
                                   dtype=torch.uint8, device=dev)
        self.result[L.RES_PENDING] = self.tokens[-1]
        self.state[L.ST_PENDING] = self.tokens[-1]
        self.state[L.ST_BASE] = len(self.tokens) - 1
        self._ev = torch.cuda.Event()
        # CUDA-graph replay on one GPU. Sharded sessions step eagerly: capturing
        # the NCCL all-gathers with the step is possible but has not been run
        # on a multi-GPU node yet, and gloo groups cannot be captured.
        self.use_graph = graph and model.world == 1
        self._graph: torch.cuda.CUDAGraph | None = None
        self._eager_steps = 0
        if prefill:
            t0 = time.perf_counter()
            self._prefill()
            torch.cuda.synchronize()
            self.wall_times["prefill"] = time.perf_counter() - t0
            self.forward_counts["prefill"] = 1

    # ------------------------------------------------------------ prefill --
    def _prefill(self) -> None:
        """Causal forward over the prompt; last_queries summed over all rows
        (engine.py:113-124)."""
        m, c = self.model, self.model.config
        P = self.prompt_len
        toks = torch.tensor(self.tokens, dtype=torch.int32, device=self.dev)
        pos = torch.arange(P, dtype=torch.int32, device=self.dev)
        q_rot = torch.empty((P, m.H, m.dh), dtype=m.dtype, device=self.dev)
        q_pre = torch.empty((c.num_layers, P, m.H, m.dh), dtype=torch.float32, device=self.dev)
        attend = m._full_attend_fn(self.full, 0, P, pos, q_rot, None)
        m.run_layers(toks, P, attend, q_pre=q_pre)
        self.q_sum.copy_(q_pre.sum(dim=1))
        del q_pre
        self.full.commit_rows(range(P))
        self.partial = self._build_partial(P - 1)

    def set_synthetic_context(self, ctx: int, seed: int = 0) -> None:
        """Bench helper: fill the full cache with `ctx` synthetic committed
        rows (K ~ N(0,1) rotated at its position, V ~ N(0,1)), a synthetic
        history / window, and rebuild the partial cache, as if `ctx` tokens
        had been generated. Data is `synthetic` in the bench line."""
        m = self.model
        if ctx + self.Tmax + self.depth > self.full.capacity:
            raise ValueError("synthetic context exceeds cache capacity")
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        F = self.full
        for l in range(m.config.num_layers):
            for h in range(m.Hk):
                kr = torch.randn((ctx, m.dh), generator=g, device=self.dev, dtype=torch.float32)
                F.k_raw[l, h, :ctx] = kr.to(m.dtype)
                half = m.dh // 2
                cs, sn = m.rope_cos[:ctx], m.rope_sin[:ctx]
                a, b = kr[:, 0::2], kr[:, 1::2]
                rot = torch.empty_like(kr)
                rot[:, 0::2] = a * cs - b * sn
                rot[:, 1::2] = a * sn + b * cs
                F.k_rot[l, h, :ctx] = rot.to(m.dtype)
                F.v[l, h, :ctx] = torch.randn((ctx, m.dh), generator=g, device=self.dev).to(m.dtype)
                del kr, rot, a, b, cs, sn, half
        F.positions = list(range(ctx))
        vocab = m.config.vocab_size
        extra = ctx + 1 - len(self.tokens)
        if extra > 0:
            synth = torch.randint(0, vocab, (extra,), generator=g, device=self.dev).cpu().tolist()
            self.tokens += synth
        self.q_sum.normal_(0.0, 1.0, generator=g)
        self.result[L.RES_PENDING] = self.tokens[-1]
        self.state[L.ST_PENDING] = self.tokens[-1]
        self.state[L.ST_BASE] = len(self.tokens) - 1
        self.partial = self._build_partial(ctx)

    # -------------------------------------------------------- partial cache --
    def _build_partial(self, upto: int) -> PartialCache:
        """engine.py:138-148: mirror below the budget, else Eq. 2 top-K. One
        GPU: one fused score -> select -> gather launch (sd_partial_refresh);
        sharded: per-head score partials all-gathered and summed in head order,
        then the same launch on the summed scores."""
        cfg, m = self.config, self.model
        part = self.partial
        if part is None:
            part = PartialCache(cfg.sink_size, cfg.budget, m.config.num_layers, m.Hk, m.dh, m.dtype, self.dev)
        if upto < cfg.budget:
            part.build_mirror(self.full, upto)
        elif m.world == 1:
            part.refresh_from(self.full, upto, q_sum=self.q_sum, num_heads=m.H)
        else:
            from .parallel import sharded_scores
            part.build_topk(self.full, sharded_scores(self.full, self.q_sum, m, cfg.sink_size, upto), upto)
        return part

    # ----------------------------------------------------------------- step --
    @property
    def done(self) -> bool:
        return len(self.emitted) >= self.config.target_length

    def _draft(self, n: int, graph: bool = False) -> None:
        """Draft forward + penalised per-head top-w + n-gram tree (engine.py:199-217).
        graph: step-invariant arguments only (whole slot range, base from state)."""
        m, cfg, smp = self.model, self.config, self.config.sampler
        part = self.partial
        q_rot, kt, vt, out = self.q_rot_d, self.kt, self.vt, self.attn_out_d
        hi = part.slot_cap  # whole slot range (holes masked): eager and replay split the draft identically

        def attend(l, qkv, q_pre):
            if qkv is not None:  # else the QKV projection already rotated and staged the row
                m.rope_stage(qkv, 1, part.count_dev(), q_rot, None, None, kt, vt, m.dh, 0)
            m.attention(q_rot, 1, 1, part.pk[l], part.pv[l], part.head_stride, hi, part.prank[l], kt, vt,
                        m.dh, None, None, out, part.tmaps, l, ws=self.attn_ws)
            return out

        pend = self.result[L.RES_PENDING:L.RES_PENDING + 1]
        h0 = m.run_layers(pend, 1, attend, rope=(part.count_dev(), q_rot, kt, vt))
        logits = m.head_logits(h0, self.depth)
        self.draft_logits = logits
        win = self.window.count if smp.window > 0 else None
        L.call("sd_draft_topw", L.ptr(logits), self.depth, m.config.vocab_size, L.ptr(win), smp.temperature,
               smp.theta, int(smp.ctrl_style), L.host_i32(cfg.tree.widths), L.ptr(self.per_head), L.stream())
        L.call("sd_draft_tree", self.ngrams.handle, cfg.k, L.ptr(self.per_head), L.host_i32(cfg.tree.widths),
               self.depth, L.ptr(self.state), -1 if graph else n - 1, L.ptr(self.grams), L.ptr(self.tree_rec),
               L.stream())

    def _verify(self, n: int, graph: bool = False) -> None:
        """Masked tree verification over the full cache + sampling + accept
        + commit + reconcile (engine.py:221-290). graph: the cache offset and
        context come from the tree record / state on device."""
        m, cfg, smp = self.model, self.config, self.config.sampler
        F = self.full
        base = n - 1
        lay = L.tree_layout()
        T = self.Tmax
        rec = self.tree_rec
        rows_dev = rec[lay["T"]:lay["T"] + 1]
        toks = rec[lay["TOK"]:lay["TOK"] + T]
        pos = rec[lay["POS"]:lay["POS"] + T]
        bits = rec[lay["MASK"]:lay["MASK"] + T * L.MASK_WORDS]
        q_rot, out = self.q_rot_v, self.attn_out_v

        if graph:
            ctx_max = F.capacity - T
            ctx_dev = pos[0:1]  # tree record POS[0] = n - 1 = live cache length

            def attend(l, qkv, q_pre):
                m.rope_stage(qkv, T, pos, q_rot, q_pre, F.k_raw[l], F.k_rot[l], F.v[l], F.head_stride, -1, rows_dev)
                m.attention(q_rot, T, 0, F.k_rot[l], F.v[l], F.head_stride, ctx_max, None, None, None,
                            F.head_stride, bits, rows_dev, out, F.tmaps, l, ctx_dev=ctx_dev, ws=self.attn_ws)
                return out
        else:
            def attend(l, qkv, q_pre):
                m.rope_stage(qkv, T, pos, q_rot, q_pre, F.k_raw[l, :, base:], F.k_rot[l, :, base:],
                             F.v[l, :, base:], F.head_stride, 0, rows_dev)
                m.attention(q_rot, T, 0, F.k_rot[l], F.v[l], F.head_stride, base, None, F.k_rot[l, :, base:],
                            F.v[l, :, base:], F.head_stride, bits, rows_dev, out, F.tmaps, l, ws=self.attn_ws)
                return out

        m.rows_hint = rows_dev  # projections skip the padded tree rows (sd_gemm_rows)
        try:
            h0 = m.run_layers(toks, T, attend, q_pre=self.q_pre)
        finally:
            m.rows_hint = None
        a = self._verify_sample_args(n, graph)
        if self._lmhead_fused(a):
            logits = self._lmhead_stats(h0, a)
        else:
            logits = m.lm_logits(h0)
        self.verify_logits = logits
        L.call("sd_sample_rows", L.ptr(logits), a, L.stream())
        L.call("sd_accept_commit", L.ptr(rec), L.ptr(self.y), self.select_seed, -1 if graph else n, self.depth,
               int(cfg.bonus), L.ptr(self.state), L.ptr(self.window.ring), L.ptr(self.window.count), smp.window,
               L.ptr(self.history), self.ngrams.handle, L.ptr(self.result), L.stream())
        F.reconcile_device(-1 if graph else base, self.result, self.q_pre, T, m.H, self.q_sum)
        # admit the accepted rows / evict to the budget (engine.py:281-283), on device
        self.partial.step_device(F, self.result)

    def _verify_sample_args(self, n: int, graph: bool) -> "L.SampleArgs":
        """Sampler arguments of the verification rows: tree-row penalty splices
        (engine.py:155-181) over the window, the configured truncation."""
        m, smp = self.model, self.config.sampler
        a = L.SampleArgs()
        a.rows, a.V, a.in_kind = self.Tmax, m.config.vocab_size, L.IN_LOGITS_F32
        _trunc_fields(a, smp)
        a.member_kind = L.MEMBER_TREE
        a.win_count, a.win_ring, a.state = L.ptr(self.window.count), L.ptr(self.window.ring), L.ptr(self.state)
        a.window = smp.window
        a.tree, a.depth = L.ptr(self.tree_rec), self.depth
        a.positions, a.n = None, -1 if graph else n
        a.token_out = L.ptr(self.y)
        return a

    def _lmhead_fused(self, a) -> bool:
        return self.model.lmhead_fused_ok(self.Tmax) and a.trunc_kind in (L.TRUNC_NONE, L.TRUNC_MIN_P, L.TRUNC_TOP_P)

    def _lmhead_stats(self, h0, a):
        """LM head + penalty + per-tile softmax statistics in one tcgen05 launch;
        `a` is switched to the sampler's scaled-input mode (engine.py:237-245)."""
        m = self.model
        if getattr(self, "_lm_bufs", None) is None:
            V, T = m.config.vocab_size, self.Tmax
            tiles = L.load().sd_lmhead_tiles(V)
            self._lm_bufs = (torch.empty((T, V), dtype=torch.float32, device=m.device),
                             torch.empty((T, tiles, 2), dtype=torch.float64, device=m.device),
                             torch.empty((T, m.config.hidden_dim), dtype=m.dtype, device=m.device), tiles)
        logits, stats, xb, tiles = self._lm_bufs
        a.in_kind, a.stats, a.stats_tiles = L.IN_LOGITS_F32, None, 0
        m.lm_head_sample_stats(h0, a, logits, stats, xb)
        a.in_kind, a.stats, a.stats_tiles = L.IN_SCALED_F32, L.ptr(stats), tiles
        return logits

    def step(self) -> IterationRecord:
        if self.done:
            raise SessionExhausted(f"{len(self.emitted)} tokens already emitted of {self.config.target_length}")
        cfg = self.config
        n = len(self.tokens)
        if n - 1 + self.depth >= self.model.config.max_positions:
            raise PositionOverflow(f"position {n - 1 + self.depth} >= max_positions {self.model.config.max_positions}")
        refreshed = needs_refresh(len(self.full), self.partial)
        if refreshed:
            self.partial = self._build_partial(len(self.full))
        t0 = time.perf_counter()
        draft_ctx = self.partial.count
        base = n - 1
        if len(self.full) > base:
            self.full.truncate(base)
        self.full.reserve(self.Tmax)
        if self.use_graph and self._eager_steps >= 1 and self._graph is None:
            try:
                self._capture()
            except Exception as e:  # noqa: BLE001 - e.g. a collective that refuses stream capture
                import warnings
                warnings.warn(f"CUDA-graph capture failed ({type(e).__name__}: {e}); running eager steps")
                torch.cuda.synchronize()
                self.use_graph = False
        if self.use_graph and self._graph is not None:
            self._graph.replay()
            L.launch_count += self._graph_launches
        else:
            self._draft(n)
            self._verify(n)
            self.result_host.copy_(self.result, non_blocking=True)
            self._eager_steps += 1
        self.forward_counts["draft"] += 1
        self.forward_counts["verify"] += 1
        t1 = time.perf_counter()
        self._ev.record()
        self._ev.synchronize()
        if self.model.world > 1:  # replicated stages stay in lock step
            from .parallel import check_lockstep
            check_lockstep(self.result, self.model.world, self.model.group, step=len(self.records))
        r = self.result_host.tolist()
        a = r[L.RES_ACCEPTED]
        ys = r[L.RES_YS:L.RES_YS + a]
        best_v, pick, origin, rows = r[L.RES_BEST], r[L.RES_PICK], r[L.RES_ORIGIN], r[L.RES_ROWS]
        pos = self.full.positions  # engine positions are range(len): trim + extend, no O(ctx) rebuild
        del pos[base:]
        pos.extend(range(base, base + a))
        self.partial.account(a)  # host mirror of the device admit/evict counters
        self.tokens.extend(ys)
        self.emitted.extend(ys)
        self.window.host_len = min(self.window.capacity, self.window.host_len + a)
        t2 = time.perf_counter()
        self.wall_times["draft"] += t1 - t0
        self.wall_times["verify"] += t2 - t1
        org = "ngram" if origin else "head"
        rec = IterationRecord(step=len(self.records), accepted=a,
                              ngram_accepted=a if (org == "ngram" and best_v == self.depth) else 0,
                              origin=org, matched=best_v, tokens=ys, forwards=2, refreshed=refreshed,
                              draft_ctx=draft_ctx, verify_ctx=base, verify_rows=rows, path_index=pick)
        self.records.append(rec)
        return rec

    # step-graph post-processing (sd_graph_relax_library_edges); A/B switch: tools only
    relax_library_edges = os.environ.get("SD_RELAX_EDGES", "1") != "0"
    relaxed_edges = 0

    def _capture(self) -> None:
        """Capture draft + verify + result copy as one CUDA graph (step-invariant
        launch arguments; see the module docstring). Capture does not run the
        work: step() replays the graph right after."""
        m, F = self.model, self.full
        torch.cuda.synchronize()
        relax = self.relax_library_edges
        g = torch.cuda.CUDAGraph(keep_graph=True) if relax else torch.cuda.CUDAGraph()
        n = len(self.tokens)
        l0 = L.launch_count
        with torch.cuda.graph(g):
            self._draft(n, graph=True)
            self._verify(n, graph=True)
            self.result_host.copy_(self.result, non_blocking=True)
        self._graph_launches = L.launch_count - l0  # our kernels per replay
        L.launch_count = l0
        if relax:
            # cuBLAS -> our kernel edges fire at the projection's launch completion
            # (our kernels wait in griddepcontrol.wait): no launch gap after cuBLAS
            import ctypes
            n_relaxed = ctypes.c_int(0)
            L.call("sd_graph_relax_library_edges", g.raw_cuda_graph(), ctypes.byref(n_relaxed))
            self.relaxed_edges = n_relaxed.value
            g.instantiate()
        self._graph = g

    def metrics(self) -> RunMetrics:
        return collect_metrics(self.records, self.gamma, self.emitted, dict(self.forward_counts),
                               dict(self.wall_times))

    def device_error(self) -> int:
        return int(self.state[L.ST_ERROR].item()) or self.partial.device_error()



def prefill(model: TinyTransformer, prompt: list[int], config: EngineConfig) -> Session:
    return Session(model, prompt, config)


def generate(model: TinyTransformer, prompt: list[int], config: EngineConfig) -> tuple[list[int], RunMetrics]:
    session = prefill(model, prompt, config)
    while not session.done:
        session.step()
    return session.emitted, session.metrics()


def generate_ar(model: TinyTransformer, prompt: list[int], config: EngineConfig) -> list[int]:
    """Plain decoding with the full cache and the same position-keyed sampler
    (engine.py:328-360): the losslessness reference."""
    config.validate(model.config.gamma)
    if len(prompt) <= config.sink_size:
        raise PromptTooShort(f"prompt length {len(prompt)} must exceed the sink size {config.sink_size}")
    smp = config.sampler
    m = model
    dev = m.device
    V = m.config.vocab_size
    cache = m.new_cache(len(prompt) + config.target_length + 8)
    P = len(prompt)
    toks = torch.tensor(prompt, dtype=torch.int32, device=dev)
    pos = torch.arange(P, dtype=torch.int32, device=dev)
    q_rot = torch.empty((P, m.H, m.dh), dtype=m.dtype, device=dev)
    h0 = m.run_layers(toks, P, m._full_attend_fn(cache, 0, P, pos, q_rot, None))
    cache.commit_rows(range(P))
    logits = m.lm_logits(h0[-1:])
    state = torch.zeros(16, dtype=torch.int64, device=dev)
    window = PenaltyWindow(smp.window, V, state=state, device=dev)
    tokens = list(prompt)
    out: list[int] = []
    tok_dev = torch.zeros(1, dtype=torch.int32, device=dev)
    pos_dev = torch.zeros(1, dtype=torch.int32, device=dev)
    q1 = torch.empty((1, m.H, m.dh), dtype=m.dtype, device=dev)
    while True:
        a = L.SampleArgs()
        a.rows, a.V, a.in_kind = 1, V, L.IN_LOGITS_F32
        _trunc_fields(a, smp)
        a.member_kind = L.MEMBER_WINDOW
        a.win_count, a.win_ring, a.state, a.window = L.ptr(window.count), L.ptr(window.ring), L.ptr(state), smp.window
        pos_dev.fill_(len(tokens))
        a.positions = L.ptr(pos_dev)
        a.token_out = L.ptr(tok_dev)
        L.call("sd_sample_rows", L.ptr(logits), a, L.stream())
        if smp.window > 0:
            L.call("sd_window_push", L.ptr(tok_dev), 1, L.ptr(state), L.ptr(window.ring), L.ptr(window.count),
                   smp.window, L.stream())
        t = int(tok_dev.item())
        out.append(t)
        tokens.append(t)
        if len(out) >= config.target_length:
            return out
        ctx = len(cache)
        pos_dev.fill_(ctx)
        h0 = m.run_layers(tok_dev, 1, m._full_attend_fn(cache, ctx, 1, pos_dev, q1, None))
        cache.commit_rows([ctx])
        logits = m.lm_logits(h0)
