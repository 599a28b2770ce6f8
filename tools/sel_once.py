"""Run the C3 selection alone a few times on uniform-random importance (for ncu
captures of k_select): python tools/sel_once.py [N] [chunk]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_02789_b200 as sp  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = torch.Generator(device="cuda").manual_seed(0)
imp = torch.rand((1, N), device="cuda", generator=g) + 1e-3
tok = torch.arange(N, dtype=torch.int32, device="cuda")[None].contiguous()
for _ in range(6):
    sp.select(imp, 0.1, 5, chunk, tokens=tok)
torch.cuda.synchronize()
print("ok")
