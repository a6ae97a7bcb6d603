"""Decode-step benchmark (driver contract; see README / DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--ctx C]

A step is one TokenSwift decode iteration (Session.step: draft forward over
the partial cache, n-gram tree, verification forward over the full cache,
sampling, acceptance, cache maintenance) of LLaMA3.1-8B-shaped random-init
weights (cfg3 of BASELINE.json) at a fixed point of a 100K-token generation
from a 4096-token prefix. Time per step is linear in the context length, so
the default point, the run's mean context (4096 + 100000/2), gives the
run-average tokens/s. The prefix is prefilled for real; the committed
context beyond it is synthetic (random K/V, `data: synthetic`).

Rank 0 prints one JSON line. --impl reference times the unmodified reference
(swiftdec, pure numpy, pip-installed into baseline/_ref; baseline/ref_arm.py)
on the host cores: cfg1 end to end, cfgs 2-5 as a bounded sample composed from
its own functions at full shape.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE_NAME = {"cfg1": "tiny LLaMA-style", "cfg2": "Qwen2.5-1.5B shape", "cfg3": "LLaMA3.1-8B shape",
              "cfg4": "YaRN-LLaMA2-7B (MHA) shape", "cfg5": "Qwen2.5-14B shape"}


def metric_name(cfg_name):
    return f"generated tokens/s (TokenSwift decode, {SHAPE_NAME[cfg_name]})"


CONFIGS = {
    # name: model dims, engine, sampler (Table 9 / SURVEY.md §8d)
    "cfg1": dict(V=32000, d=256, L=2, H=8, Hk=2, prefix=512, gen=2000, B=512, S=32, trunc=("min_p", 1.0), theta=1.2),
    "cfg2": dict(V=151936, d=1536, L=28, H=12, Hk=2, prefix=2048, gen=20000, B=2048, S=32, trunc=("top_p", 0.9),
                 theta=1.15),
    "cfg3": dict(V=128256, d=4096, L=32, H=32, Hk=8, prefix=4096, gen=100000, B=4096, S=32, trunc=("min_p", 0.1),
                 theta=1.2),
    "cfg4": dict(V=32000, d=4096, L=32, H=32, Hk=32, prefix=4096, gen=100000, B=4096, S=32, trunc=("top_p", 0.9),
                 theta=1.15),
    "cfg5": dict(V=152064, d=5120, L=48, H=40, Hk=8, prefix=4096, gen=100000, B=4096, S=32, trunc=("min_p", 0.05),
                 theta=1.13),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--ctx", type=int, default=None, help="committed context at the timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--attn-reps", type=int, default=3)
    ap.add_argument("--ngram-stress", action="store_true",
                    help="SURVEY §8d stress line: before the timed steps, seed the n-gram table with k=20 unique "
                         "frequent branches from the draft's first token, so every tree has 1+40+60 = 101 rows")
    return ap.parse_args()


def workload_name(cfg_name, c, ctx):
    return (f"{cfg_name}: TokenSwift decode step, random-init {c['L']}L d={c['d']} H={c['H']} Hk={c['Hk']} "
            f"V={c['V']} (reference arch), tree [1,3,3,3] + k=20 n-grams, partial budget {c['B']} sink {c['S']}, "
            f"prefix {c['prefix']} prefilled, generation of {c['gen']} at mean context ctx={ctx}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    nvidia-smi takes ~0.1-0.3 s to start, so the sampler is started before the
    warm-up (start()) and only the samples whose timestamps fall inside the
    timed window (mark_begin() / mark_end()) are summarised."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.t_begin = self.t_end = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def mark_begin(self):
        self.t_begin = time.time()

    def mark_end(self):
        self.t_end = time.time()
        time.sleep(0.1)  # let the sampler flush the window's last samples
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        import datetime
        sm, mx, power, reasons, n_all = [], 0, [], set(), 0
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, cmax = float(f[2]), float(f[3])
            except (ValueError, IndexError):
                continue
            n_all += 1
            if self.t_begin is not None and not (self.t_begin - 0.01 <= ts <= (self.t_end or ts) + 0.01):
                continue
            sm.append(clk)
            mx = max(mx, cmax)
            try:
                power.append(float(f[4]))
            except ValueError:
                pass
            for i, n in enumerate(self.NAMES):
                if len(f) > 6 + i and f[6 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "sm_min_mhz": min(sm) if sm else None, "power_w": statistics.median(power) if power else None,
                "reasons": sorted(reasons), "samples": len(sm), "samples_total": n_all}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic():
    """dram__bytes_read + dram__bytes_write per launch of the verification kernel
    from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_verify_traffic.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get("traffic_bytes_per_launch")


def cpu_baseline_line(c, ctx, accepted, tree_rows, samples=2):
    """The unmodified reference's CPU path on the host cores, composed from its
    own functions at full shape (baseline/ref_arm.py; kind "reference"); the
    oracle port (kind "port") when the reference cannot be imported."""
    from baseline import ref_arm
    if ref_arm.import_reference()[0] is not None:
        comp = ref_arm.Composer(c, ctx, rows=tree_rows)
        per = [comp.sample(accepted)[0] for _ in range(samples + 1)][1:]  # first sample warms
        it = statistics.median(per)
        return {"value": accepted / it, "unit": "tokens/s", "cores": ref_arm.host_cores(), "kind": "reference",
                "composed": True,
                "sample": (f"reference swiftdec functions at full shape, composed per iteration ({c['L']} x verify "
                           f"layer over ctx {ctx} with {tree_rows} rows + draft + cache maintenance + sampling + "
                           f"top-w + n-gram/tree + amortised refresh); {accepted:.2f} tokens/iteration; "
                           f"{it:.1f} s/iteration; median of {samples} samples")}
    from oracle.cpu_baseline import compose_step, host_cores
    per_step, tps, parts = compose_step(c["d"], c["L"], c["H"], c["Hk"], c["V"], ctx, c["B"], tree_rows=tree_rows,
                                        accepted=accepted)
    return {"value": tps, "unit": "tokens/s", "cores": host_cores(), "kind": "port",
            "sample": (f"oracle (numpy fp64) pieces at full shape, composed: {c['L']} x (1 verify layer, "
                       f"{tree_rows} rows over ctx {ctx} + 1 draft layer over {c['B']}) + LM head (1/16 vocab "
                       f"slice x16) + sampling {tree_rows}x{c['V']} + tree/n-gram/accept; "
                       f"{accepted:.2f} tokens/step; {per_step:.1f} s/step"),
            "parts_s": {k: round(v, 4) for k, v in parts.items()}}


def run_reference(args, c, ctx):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the unmodified reference (baseline/_ref or /root/reference): cfg1 end to
    # end, cfgs 2-5 composed from its own functions at full shape
    from baseline import ref_arm
    if ref_arm.run(args, c, ctx, metric_name(args.config), workload_name(args.config, c, ctx)) is not None:
        return
    # reference not importable here: the oracle port, composed (kind "port")
    steps, warm = max(1, min(args.steps, 2)), 0
    vals = []
    for _ in range(steps):
        line = cpu_baseline_line(c, ctx, accepted=4.0, tree_rows=41)
        vals.append(line["value"])
    v = statistics.median(vals)
    out = {"metric": metric_name(args.config), "value": v, "unit": "tokens/s",
           "impl": "reference", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
           "ms_per_step": 4000.0 / v if v else None, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(args.config, c, ctx), "ctx": ctx},
           "cpu_baseline": {**line, "value": v},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    c = CONFIGS[args.config]
    ctx = args.ctx if args.ctx is not None else c["prefix"] + c["gen"] // 2
    if args.impl == "reference":
        run_reference(args, c, ctx)
        return
    import torch
    import torch.distributed as dist

    import paper_2502_18890_b200 as sd
    from paper_2502_18890_b200 import _lib
    from paper_2502_18890_b200.parallel import init_from_env

    rank, world, local = init_from_env("nccl")
    torch.cuda.set_device(local)
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    maxpos = c["prefix"] + c["gen"] + 256
    mcfg = sd.ModelConfig(vocab_size=c["V"], num_layers=c["L"], hidden_dim=c["d"], num_heads=c["H"],
                          num_kv_heads=c["Hk"], gamma=3, max_positions=maxpos, init_seed=0)
    model = sd.TinyTransformer(mcfg, dtype=torch.bfloat16, init="device", shard=(rank, world),
                               group=None)
    trunc = sd.Truncation(*c["trunc"])
    ecfg = sd.EngineConfig(target_length=c["gen"], sink_size=c["S"], budget=c["B"], tree=sd.TreeConfig((1, 3, 3, 3)),
                           k=20, sampler=sd.SamplerConfig(theta=c["theta"], window=1024, truncation=trunc))
    prompt = sd.rng.random_prompt(c["prefix"], c["V"])
    t0 = time.perf_counter()
    sess = sd.Session(model, prompt, ecfg, capacity=c["prefix"] + c["gen"] + 512)
    prefill_s = time.perf_counter() - t0
    if ctx > c["prefix"]:
        sess.set_synthetic_context(ctx)
    torch.cuda.synchronize()
    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        sess.step()
    if args.ngram_stress:
        seed_unique_ngrams(sess, model, c)
        for _ in range(2):
            sess.step()
    # ---- timed region: device time (events on the launching stream), max over ranks ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = len(sess.records)
    l0 = _lib.launch_count
    clk.mark_begin()
    torch.cuda.nvtx.range_push("timed")
    w0 = time.perf_counter()
    e0.record(st)
    for _ in range(args.steps):
        sess.step()  # public API: includes the per-step D2H of the step result
    e1.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    torch.cuda.nvtx.range_pop()
    clk.mark_end()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count - l0
    recs = sess.records[n0:]
    tokens = sum(r.accepted for r in recs)
    dev_s = e0.elapsed_time(e1) / 1e3
    t = torch.tensor([dev_s, wall], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, wall = float(t[0]), float(t[1])
    # ---- dominant kernel: verification attention, timed alone per layer ----
    rows = max(1, round(statistics.mean(r.verify_rows for r in recs)))
    hbm, tflops, peak_kind = measured_peaks()
    attn = time_verify_attention(sess, model, rows, ctx, reps=args.attn_reps)
    dh, Hk, H = model.dh, model.Hk, model.H
    alg_bytes = 2 * ctx * Hk * dh * 2 + 2 * rows * H * dh * 2 + 2 * rows * Hk * dh * 2
    alg_flops = 4 * rows * H * dh * ctx
    achieved = alg_bytes / attn["avg_s"] / 1e9
    bound = "hbm" if (alg_flops / (tflops * 1e12)) < (alg_bytes / (hbm * 1e9)) else "tensor"
    kernels = {"draft_attention": time_draft_attention(sess, model, hbm, reps=args.attn_reps)}
    relaxed_edges = getattr(sess, "relaxed_edges", 0)
    lm = time_lmhead(sess, model, hbm, reps=args.attn_reps)
    if lm is not None:
        kernels["lm_head"] = lm
    if world == 1:
        kernels["refresh"] = time_refresh(sess, model, ctx, hbm, reps=args.attn_reps)
        acc = tokens / max(1, len(recs))
        kernels["refresh"]["amortised_ms_per_step"] = (kernels["refresh"]["avg_launch_us"] / 1e3 * acc
                                                       / (c["B"] - c["S"] + 1))
    if rank != 0:
        if world > 1:
            dist.barrier()
        return
    clocks = clk.summary()
    out = {
        "metric": metric_name(args.config),
        "value": tokens / dev_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights; random prompt prefilled; synthetic KV beyond the prefix)",
        "config": {"workload": workload_name(args.config, c, ctx) + (" (n-gram stress: 101-row trees)"
                                                                     if args.ngram_stress else ""),
                   "ctx": ctx, "global_batch": 1,
                   "parallelism": f"kv-head shard x{world}", "l2": "inputs larger than L2 (12.4 GB weights + KV per step)"},
        "e2e": {"value": tokens / wall, "unit": "tokens/s", "h2d_bytes_per_step": 4, "d2h_bytes_per_step": 128,
                "note": "Session.step() wall clock incl. per-step result D2H"},
        "gpu_launches": launches,
        "graph_relaxed_edges": relaxed_edges,
        "roofline": {"bound": bound, "achieved": achieved if bound == "hbm" else alg_flops / attn["avg_s"] / 1e12,
                     "peak": hbm if bound == "hbm" else tflops, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
                     "frac": (achieved / hbm) if bound == "hbm" else (alg_flops / attn["avg_s"] / 1e12) / tflops,
                     "traffic": ncu_traffic(), "kernel": "sd_attention verify (tcgen05 split-KV + merge), one layer",
                     "peak_kind": peak_kind, "alg_bytes_per_launch": alg_bytes, "alg_flops_per_launch": alg_flops,
                     "avg_launch_us": attn["avg_s"] * 1e6, "rows": rows,
                     "share_of_step": attn["avg_s"] * model.config.num_layers / (dev_s / args.steps)},
        "kernels": kernels,
        "clocks": clocks,
        "alpha": statistics.mean(r.accepted for r in recs) / 4.0,
        "mean_verify_rows": statistics.mean(r.verify_rows for r in recs),
        "iterations_per_s": args.steps / dev_s, "prefill_s": prefill_s,
        "refreshes": sum(r.refreshed for r in recs),
    }
    if not args.no_cpu_baseline and world == 1:
        mean_acc = tokens / max(1, len(recs))
        out["cpu_baseline"] = cpu_baseline_line(c, ctx, accepted=mean_acc, tree_rows=rows)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()


def seed_unique_ngrams(sess, model, c, k=20, weight=64):
    """Insert k grams (x, a, b, c) with random continuations, each counted
    `weight` times, for the draft's likely first token x (random-init weights
    repeat one token, so x is the last emitted token): retrieval then returns
    k unique chains that do not merge with the head trie, and the verify tree
    has its maximum 1 + 40 + 3k rows."""
    import torch
    g = torch.Generator()
    g.manual_seed(7)
    x = sess.emitted[-1] if sess.emitted else sess.tokens[-1]
    for i in range(k):
        tail = torch.randint(0, c["V"], (3,), generator=g).tolist()
        for _ in range(weight):
            sess.ngrams.update([x] + tail, [])


def time_verify_attention(sess, model, rows, ctx, reps=3):
    """CUDA-event time of the verification attention alone (tcgen05 kernel +
    split merge), one launch per layer (each layer's K/V is a distinct >L2
    buffer), captured in a CUDA graph and replayed on the launching stream, so
    the host's per-call overhead (~30 us of Python + ctypes, which would floor
    small-context shapes) is not in the number."""
    import torch
    F = sess.full
    T = rows
    q = torch.randn((T, model.H, model.dh), device="cuda").mul_(0.1).to(model.dtype)
    out = torch.empty((T, model.H * model.dh), dtype=model.dtype, device="cuda")
    from paper_2502_18890_b200 import _lib as L
    from paper_2502_18890_b200.model import mask_bits_from_bool
    import numpy as np
    m = np.tril(np.ones((T, T), dtype=bool))
    bits = torch.as_tensor(mask_bits_from_bool(m), device="cuda")
    base = min(ctx, len(F))
    ws = torch.zeros(L.load().sd_attention_workspace_bytes(T, model.H, model.dh, base), dtype=torch.uint8,
                     device="cuda")
    Ln = model.config.num_layers

    def layers():
        for l in range(Ln):
            model.attention(q, T, 0, F.k_rot[l], F.v[l], F.head_stride, base, None, F.k_rot[l, :, base:],
                            F.v[l, :, base:], F.head_stride, bits, None, out, F.tmaps, l, ws=ws)
    avg = _graph_time(layers, reps) / Ln
    return {"avg_s": avg, "launches": reps * Ln}


def time_refresh(sess, model, ctx, hbm, reps=3):
    """CUDA-event time of one partial-cache refresh at the bench context (the
    fused score -> top-K -> gather launch, all layers; engine.py:150-151,
    kvcache.py:243-297), on the launching stream. Algorithmic bytes per layer
    (SURVEY §8d): score (ctx-S)*Hk*dh*2 + (ctx-S)*4, select + gather
    (ctx-S)*4 + 2*(B-S)*Hk*dh*2*2."""
    import torch
    part, cfg = sess.partial, sess.config
    st = torch.cuda.current_stream()
    part.refresh_from(sess.full, ctx, q_sum=sess.q_sum, num_heads=model.H)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        part.refresh_from(sess.full, ctx, q_sum=sess.q_sum, num_heads=model.H)
    e1.record(st)
    torch.cuda.synchronize()
    avg = e0.elapsed_time(e1) / 1e3 / reps
    S, B, Hk, dh, Ln = cfg.sink_size, cfg.budget, model.Hk, model.dh, model.config.num_layers
    n = ctx - S
    alg = Ln * (n * Hk * dh * 2 + n * 4 + n * 4 + 2 * (B - S) * Hk * dh * 2 * 2)
    return {"bound": "hbm", "achieved": alg / avg / 1e9, "peak": hbm, "unit": "GB/s", "frac": alg / avg / 1e9 / hbm,
            "avg_launch_us": avg * 1e6, "alg_bytes_per_launch": alg, "ctx": ctx, "layers": Ln,
            "kernel": "sd_partial_refresh (fused Eq. 2 score -> radix top-K -> gather -> importance ring), all layers"}


def _graph_time(fn, reps):
    """Seconds per call of fn() (a run of kernel launches), captured once in a
    CUDA graph and replayed `reps` times between CUDA events on the replay
    stream: device time without the host's per-launch overhead."""
    import torch
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()  # warm on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def time_lmhead(sess, model, hbm, reps=3):
    """CUDA-event time of the fused verification LM head (sd_lmhead_sample_stats:
    embedding stream + penalty + scaled logits + tile statistics) with the
    session's own arguments and buffers, 4 launches back to back per replay."""
    import torch
    a = sess._verify_sample_args(0, True)
    if not sess._lmhead_fused(a):
        return None
    T, V, d = sess.Tmax, model.config.vocab_size, model.config.hidden_dim
    h0 = torch.randn((T, d), device="cuda")

    def one():
        sess._lmhead_stats(h0, sess._verify_sample_args(0, True))
    avg = _graph_time(lambda: [one() for _ in range(4)], reps) / 4
    live = int(sess.tree_rec[0].item())
    tiles = (V + 127) // 128
    alg = V * d * 2 + T * d * 2 + live * V * 4 + live * tiles * 16
    return {"bound": "hbm", "achieved": alg / avg / 1e9, "peak": hbm, "unit": "GB/s", "frac": alg / avg / 1e9 / hbm,
            "avg_launch_us": avg * 1e6, "alg_bytes_per_launch": alg, "rows": live,
            "kernel": "sd_lmhead_sample_stats (tcgen05 tied LM head + penalty + scaled logits + tile softmax stats)"}


def time_draft_attention(sess, model, hbm, reps=3):
    """CUDA-event time of the draft attention alone (the step's own call: whole
    slot range, rank-RoPE, fused merge), one launch per layer, back to back."""
    import torch
    part = sess.partial
    q = torch.randn((1, model.H, model.dh), device="cuda").mul_(0.1).to(model.dtype)
    out = torch.empty((1, model.H * model.dh), dtype=model.dtype, device="cuda")
    kt = torch.randn((model.Hk, model.dh), device="cuda").to(model.dtype)
    vt = torch.randn_like(kt)
    hi = part.slot_cap

    def one(l):
        model.attention(q, 1, 1, part.pk[l], part.pv[l], part.head_stride, hi, part.prank[l], kt, vt, model.dh,
                        None, None, out, part.tmaps, l, ws=sess.attn_ws)
    avg = _graph_time(lambda: [one(l) for l in range(model.config.num_layers)], reps) / model.config.num_layers
    m = part.count
    alg = 2 * (m + 1) * model.Hk * model.dh * 2 + 2 * model.H * model.dh * 2
    return {"bound": "hbm", "achieved": alg / avg / 1e9, "peak": hbm, "unit": "GB/s", "frac": alg / avg / 1e9 / hbm,
            "avg_launch_us": avg * 1e6, "alg_bytes_per_launch": alg, "live_slots": m, "slot_range": hi,
            "kernel": "sd_attention draft (tensor-core, rank-RoPE, fused merge), one layer"}


if __name__ == "__main__":
    main()
