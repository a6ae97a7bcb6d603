"""How much faster are the decode GEMMs when their weights are already in L2?
(cold: weights rotated over > L2 copies; warm: the same weights re-read)."""
import torch
dev = "cuda"
for M in (1, 101):
    for name, (K, N) in {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 16384)}.items():
        copies = max(2, int(600e6 // (K * N * 2)))
        Ws = [(torch.randn(K, N, device=dev) * 0.02).to(torch.bfloat16) for _ in range(copies)]
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        res = []
        for mode in ("cold", "warm"):
            def run(i):
                w = Ws[i % copies] if mode == "cold" else Ws[0]
                return torch.mm(x, w, out_dtype=torch.float32)
            for i in range(5):
                run(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(40):
                run(i)
            e1.record()
            torch.cuda.synchronize()
            res.append(f"{mode} {e0.elapsed_time(e1) / 40 * 1e3:6.1f} us")
        print(f"M={M:3d} {name}: " + " | ".join(res), flush=True)
