"""Golden end-to-end run of the REFERENCE at BASELINE cfg1 (SURVEY §8(c)
layering (3), verdict r1): V=32000, d=256, 2 layers, 8 heads, 2 kv heads,
prefix 512 (the reference's seeded random prompt), 2000 generated tokens,
budget 512, sink 32, greedy (min-p 1.0), theta 1.2, window 1024, tree
[1,3,3,3], k=20 — the emitted tokens, every IterationRecord, and the
autoregressive tokens of generate_ar (losslessness).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cfg1.py   # ~6 min on 8 cores

Writes tests/golden/cfg1_run.json; nothing at test time reads /root/reference.
"""
import json
import os
import sys
import time

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import swiftdec as S  # noqa: E402
from swiftdec.rng import derive_seed, mix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MCFG = dict(vocab_size=32000, num_layers=2, hidden_dim=256, num_heads=8, num_kv_heads=2, gamma=3,
            max_positions=4096, init_seed=0)
ENG = dict(target_length=2000, sink_size=32, budget=512, k=20)


def main():
    model = S.TinyTransformer(S.ModelConfig(**MCFG))
    seed = derive_seed(0, "prompt")
    prompt = [mix(seed, i) % MCFG["vocab_size"] for i in range(512)]
    smp = S.SamplerConfig(theta=1.2, window=1024, truncation=S.Truncation.min_p(1.0))
    cfg = S.EngineConfig(tree=S.TreeConfig((1, 3, 3, 3)), sampler=smp, **ENG)
    t0 = time.time()
    sess = S.prefill(model, prompt, cfg)
    while not sess.done:
        sess.step()
    t_swift = time.time() - t0
    t0 = time.time()
    ar = S.generate_ar(model, prompt, cfg)
    t_ar = time.time() - t0
    recs = [json.loads(r.to_json()) for r in sess.records]
    out = {"model": MCFG, "engine": ENG, "sampler": {"theta": 1.2, "window": 1024, "min_p": 1.0},
           "prompt_len": 512, "emitted": sess.emitted, "records": recs, "ar": ar,
           "lossless": ar == sess.emitted[:len(ar)], "swift_s": t_swift, "ar_s": t_ar}
    with open(os.path.join(HERE, "cfg1_run.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"cfg1: {len(sess.emitted)} tokens in {len(recs)} iterations ({t_swift:.0f} s), "
          f"refreshes {sum(r['refreshed'] for r in recs)}, AR lossless {out['lossless']} ({t_ar:.0f} s)")


if __name__ == "__main__":
    main()
