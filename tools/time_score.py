"""Time sp_score (fused) on an 8B-geometry prompt of N tokens: python tools/time_score.py N [N ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402

for n in [int(x) for x in sys.argv[1:]]:
    w = gen.CONFIGS["C3"].with_(N=n)
    Q, K, T = spgen_cuda.make_inputs(w)
    out = torch.empty((1, n), dtype=torch.float32, device="cuda")
    for _ in range(5):
        sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=out, algo="fused")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()                       # 20 launches, no host overhead in the timing
    with torch.cuda.graph(g):
        for _ in range(20):
            sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=out, algo="fused")
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"N={n}: {ms:.4f} ms  {w.k_bytes / ms / 1e6:.0f} GB/s  plan {sp.score_plan(Q, K, w.Rv)}")
    del Q, K, T
