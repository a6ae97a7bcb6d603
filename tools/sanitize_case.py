"""Small product-shape decode for compute-sanitizer (racecheck / synccheck /
memcheck): bf16, head_dim 128 (tcgen05 verification attention, tensor-core
draft attention with its fused split merge, TMA-ring gemv, cluster sampler and
top-w, fused refresh with its cluster select, in-graph admit/evict), a prompt
longer than the budget so refreshes run, eager steps then CUDA-graph replays.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18890_b200 as sd  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mcfg = sd.ModelConfig(vocab_size=4096, num_layers=2, hidden_dim=1024, num_heads=8, num_kv_heads=2, gamma=3,
                      max_positions=2048, init_seed=0)
m = sd.TinyTransformer(mcfg, dtype=torch.bfloat16, init="device")
smp = sd.SamplerConfig(theta=1.2, window=1024, truncation=sd.Truncation.min_p(0.1))
cfg = sd.EngineConfig(target_length=4 * steps + 8, sink_size=16, budget=96, tree=sd.TreeConfig((1, 3, 3, 3)), k=20,
                      sampler=smp)
s = sd.Session(m, sd.rng.random_prompt(300, mcfg.vocab_size), cfg)
for _ in range(steps):
    if s.done:
        break
    s.step()
torch.cuda.synchronize()
print(f"sanitize case ok: {len(s.emitted)} tokens, {len(s.records)} iterations, "
      f"refreshes={sum(r.refreshed for r in s.records)}, graph={s._graph is not None}, err={s.device_error()}")
