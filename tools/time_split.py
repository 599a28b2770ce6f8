"""Time the split API on one GPU: sp_score_stats, sp_score_finish (lse given --
also the row-f2 hand-over) and sp_score, for a config (debug tool)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402


def timed(fn, n=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


w = gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
Q, K, T = spgen_cuda.make_inputs(w)
stats = sp.score_stats(Q, K, w.Rv, w.scale)
lse2 = sp.stats_combine(stats[None].contiguous())
kb = K.numel() * 2 / 1e9
for name, fn in [("score (fused)", lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")),
                 ("score_stats", lambda: sp.score_stats(Q, K, w.Rv, w.scale)),
                 ("score_finish", lambda: sp.score_finish(Q, K, lse2, w.Rv, w.scale))]:
    ms = timed(fn)
    print(f"{w.name} {name:14s} {ms:.4f} ms  {kb / ms:.2f} TB/s of K")

# row f1: one rank's share of a P-way head split (the rest is an all-reduce of 4*Rv B/token)
for P in (2, 8):
    n = w.Hkv // P
    Qh, Kh = Q[:, :, :, :n * w.G], K[:, :, :n]
    acc = sp.score_acc(Qh, Kh, w.Rv, w.scale)
    ms = timed(lambda: sp.score_acc(Qh, Kh, w.Rv, w.scale, out=acc))
    print(f"{w.name} score_acc 1/{P} heads {ms:.4f} ms  {kb / P / ms:.2f} TB/s of K  (all-reduce {acc.numel() * 4 / 1e6:.1f} MB)")
