"""A real 100K-token TokenSwift generation on one B200 (cfg3 of BASELINE.json:
LLaMA3.1-8B-shaped random-init weights, reference architecture, prefix 4096,
tree [1,3,3,3], k=20, partial budget 4096 / sink 32, min-p 0.1, theta 1.2)
through the public Session.step() loop (what generate() runs), no synthetic
context: every one of the ~25K iterations drafts, verifies, samples, commits,
admits/evicts and refreshes for real.

Reports device tokens/s over the decode (CUDA events around the loop, prefill
excluded), wall tokens/s, alpha, mean verify rows, refresh count, peak
context, and a timeline (every --every iterations: context, ms/iteration).

    python tools/run_100k.py [--gen 100000] [--config cfg3] [--out profiles/r02_run_100k.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2502_18890_b200 as sd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--gen", type=int, default=None)
ap.add_argument("--every", type=int, default=1000)
ap.add_argument("--out", default=None)
args = ap.parse_args()
c = bench.CONFIGS[args.config]
gen = args.gen or c["gen"]
mcfg = sd.ModelConfig(vocab_size=c["V"], num_layers=c["L"], hidden_dim=c["d"], num_heads=c["H"], num_kv_heads=c["Hk"],
                      gamma=3, max_positions=c["prefix"] + gen + 256, init_seed=0)
model = sd.TinyTransformer(mcfg, dtype=torch.bfloat16, init="device")
ecfg = sd.EngineConfig(target_length=gen, sink_size=c["S"], budget=c["B"], tree=sd.TreeConfig((1, 3, 3, 3)), k=20,
                       sampler=sd.SamplerConfig(theta=c["theta"], window=1024, truncation=sd.Truncation(*c["trunc"])))
prompt = sd.rng.random_prompt(c["prefix"], c["V"])
t0 = time.perf_counter()
sess = sd.Session(model, prompt, ecfg, capacity=c["prefix"] + gen + 512)
prefill_s = time.perf_counter() - t0
st = torch.cuda.current_stream()
ev0 = torch.cuda.Event(enable_timing=True)
ev0.record(st)
w0 = time.perf_counter()
marks = []  # (iteration, tokens, ctx, event)
last = (0, 0)
while not sess.done:
    sess.step()
    it = len(sess.records)
    if it % args.every == 0:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        marks.append((it, len(sess.emitted), sess.records[-1].verify_ctx, e))
ev1 = torch.cuda.Event(enable_timing=True)
ev1.record(st)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
dev = ev0.elapsed_time(ev1) / 1e3
recs = sess.records
timeline, prev_t, prev_it = [], 0.0, 0
for it, toks, ctx, e in marks:
    t = ev0.elapsed_time(e) / 1e3
    timeline.append({"iteration": it, "tokens": toks, "ctx": ctx,
                     "ms_per_iteration": (t - prev_t) * 1e3 / max(1, it - prev_it)})
    prev_t, prev_it = t, it
n_tok = len(sess.emitted)
out = {
    "workload": bench.workload_name(args.config, c, None).replace(" at mean context ctx=None", "") + " (real run)",
    "generated_tokens": n_tok, "iterations": len(recs),
    "device_tokens_per_s": n_tok / dev, "wall_tokens_per_s": n_tok / wall, "decode_device_s": dev, "decode_wall_s": wall,
    "prefill_s": prefill_s, "alpha": sess.metrics().alpha,
    "mean_verify_rows": statistics.mean(r.verify_rows for r in recs),
    "max_verify_rows": max(r.verify_rows for r in recs),
    "refreshes": sum(r.refreshed for r in recs), "peak_ctx": max(r.verify_ctx for r in recs),
    "ngram_table_entries": len(sess.ngrams), "device_error": sess.device_error(),
    "timeline": timeline,
}
s = json.dumps(out)
print(s)
if args.out:
    with open(args.out, "w") as fh:
        fh.write(json.dumps(out, indent=1) + "\n")
