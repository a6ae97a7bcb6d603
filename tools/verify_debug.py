"""Debug: one verify-attention call at a small shape (tcgen05 path), synchronised."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.verify_bench import call, setup  # noqa: E402

ctx, T, T_host, Hk, G = [int(x) for x in (sys.argv[1:] or ["5000", "41", "101", "8", "4"])]
S = setup(ctx, T_host, Hk, G)
rows = torch.tensor([T], dtype=torch.int32, device="cuda")
call(S, ctx, T_host, Hk, rows_dev=rows if T != T_host else None)
torch.cuda.synchronize()
print("ok")
