import sys, torch
sys.path.insert(0, ".")
import paper_2502_18890_b200 as sd
from paper_2502_18890_b200 import _lib as L
mcfg = sd.ModelConfig(vocab_size=152064, num_layers=2, hidden_dim=5120, num_heads=40, num_kv_heads=8, gamma=3,
                      max_positions=8192, init_seed=0)
m = sd.TinyTransformer(mcfg, dtype=torch.bfloat16, init="device")
ecfg = sd.EngineConfig(target_length=64, sink_size=32, budget=512, tree=sd.TreeConfig((1, 3, 3, 3)), k=20,
                       sampler=sd.SamplerConfig(theta=1.13, window=1024, truncation=sd.Truncation.min_p(0.05)))
prompt = sd.rng.random_prompt(600, 152064)
s = sd.Session(m, prompt, ecfg, graph=False)
torch.cuda.synchronize()
print("prefill ok")
n = len(s.tokens)
s.draft_pos.fill_(s.partial.count)
s._draft(n)
torch.cuda.synchronize()
lg = s.draft_logits
print("draft logits finite:", bool(torch.isfinite(lg).all()), lg.shape, "per_head", s.per_head.tolist())
# check gemv vs mm on the first layer weights
ly = m.layers[0]
x = torch.randn(1, 5120, device="cuda").to(torch.bfloat16)
for key in ("wqkv", "wo", "w1", "w2"):
    w = ly[key]
    xx = torch.randn(1, w.shape[0], device="cuda").to(torch.bfloat16)
    a = m.gemv(xx, w)
    b = xx.float() @ w.float()
    print(key, tuple(w.shape), "max err", float((a - b).abs().max()), "finite", bool(torch.isfinite(a).all()))
