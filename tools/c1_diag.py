"""Small-prompt diagnosis (C1 and every per-rank shard of the sequence split):
graph-timed fused score, statistics-only and finish (lse given) launches over a
range of prompt lengths, forced plans at 4K, and the read-only stream probe at
the same byte counts -- separates the fixed per-launch cost, the streaming rate
and the cost of the coupled statistics exchange.  Debug tool (GPU)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402


def gtime(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        best = ms if best is None else min(best, ms)
    return best


Ns = [int(x) for x in os.environ.get("DIAG_NS", "512,1024,2048,4096,8192,16384").split(",")]
plans = [p for p in os.environ.get("DIAG_PLANS", "").split(";") if p]
for n in Ns:
    w = gen.CONFIGS["C3"].with_(N=n)
    Q, K, T = spgen_cuda.make_inputs(w)
    out = torch.empty((1, n), dtype=torch.float32, device="cuda")
    gb = w.k_bytes / 1e9
    ms_f = gtime(lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=out, algo="fused"))
    st = sp.score_stats(Q, K, w.Rv, w.scale)
    lse2 = sp.stats_combine(st[None].contiguous())
    ms_s = gtime(lambda: sp.score_stats(Q, K, w.Rv, w.scale, out=st))
    ms_fi = gtime(lambda: sp.score_finish(Q, K, lse2, w.Rv, w.scale, out=out))
    rs = spgen_cuda.read_stream_gbs(torch.device("cuda"), nbytes=max(w.k_bytes, 1 << 24), reps=10)
    print(f"N={n:6d} K={gb * 1e3:8.1f} MB  fused {ms_f * 1e3:8.1f} us ({gb / ms_f:.2f} TB/s)  "
          f"stats {ms_s * 1e3:8.1f} us  finish {ms_fi * 1e3:8.1f} us  "
          f"probe tma {w.k_bytes / rs['tma_bulk'] / 1e3:8.1f} us ld {w.k_bytes / rs['ld_v4'] / 1e3:8.1f} us  "
          f"plan {sp.score_plan(Q, K, w.Rv)}", flush=True)
    if n == 4096:
        for pstr in plans:
            os.environ["SP_FUSED_PLAN"] = pstr
            ms = gtime(lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=out, algo="fused"))
            pl = sp.score_plan(Q, K, w.Rv)
            print(f"   plan {pstr:10s} {ms * 1e3:8.1f} us  {gb / ms:.2f} TB/s  {pl}", flush=True)
        os.environ.pop("SP_FUSED_PLAN", None)
    del Q, K, T
