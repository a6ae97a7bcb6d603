"""KV-head-sharded decode on ONE GPU: two ranks (gloo, both on cuda:0) run the
sharded session and rank 0 compares the emitted tokens and records with an
unsharded session of the same weights. Exercises the all-gather of attention
outputs, the head-ordered score exchange at refresh and the replicated
sampling / tree / acceptance of parallel.py end to end.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tools/mp_sharded_check.py
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18890_b200 as sd  # noqa: E402
from paper_2502_18890_b200.parallel import init_from_env  # noqa: E402

rank, world, _ = init_from_env("gloo")
torch.cuda.set_device(0)
# --bf16: the product precision and head size (bf16, head_dim 128: tcgen05
# verification attention with model-wide split counts, tensor-core draft
# attention, fused refresh on all-gathered head-ordered scores)
BF16 = "--bf16" in sys.argv
if BF16:
    mcfg = sd.ModelConfig(vocab_size=2048, num_layers=2, hidden_dim=1024, num_heads=8, num_kv_heads=2, gamma=3,
                          max_positions=4096, init_seed=3)
    dtype, plen, target, budget = torch.bfloat16, 600, 200, 160
else:
    mcfg = sd.ModelConfig(vocab_size=512, num_layers=2, hidden_dim=256, num_heads=8, num_kv_heads=2, gamma=3,
                          init_seed=3)
    dtype, plen, target, budget = torch.float32, 80, 160, 64
cfg = sd.EngineConfig(target_length=target, sink_size=8, budget=budget, tree=sd.TreeConfig((1, 3, 3, 3)), k=20,
                      sampler=sd.SamplerConfig(theta=1.2, window=256, truncation=sd.Truncation.min_p(0.5)))
prompt = sd.rng.random_prompt(plen, mcfg.vocab_size)
m = sd.TinyTransformer(mcfg, dtype=dtype, shard=(rank, world))
s = sd.Session(m, prompt, cfg)
recs = []
while not s.done:
    r = s.step()
    recs.append((r.accepted, r.refreshed, list(r.tokens)))
if rank == 0:
    ref_m = sd.TinyTransformer(mcfg, dtype=dtype)
    ref = sd.Session(ref_m, prompt, cfg, graph=False)
    ref_recs = []
    while not ref.done:
        r = ref.step()
        ref_recs.append((r.accepted, r.refreshed, list(r.tokens)))
    same = s.emitted == ref.emitted and recs == ref_recs
    print(f"sharded x{world} ({dtype}): {len(s.emitted)} tokens, {sum(r[1] for r in recs)} refreshes; "
          f"identical to unsharded: {same}", flush=True)
    if not same:
        i = next((j for j in range(min(len(s.emitted), len(ref.emitted))) if s.emitted[j] != ref.emitted[j]), None)
        print("first token divergence at", i)
dist.barrier()
dist.destroy_process_group()
