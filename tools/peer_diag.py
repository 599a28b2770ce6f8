"""Diagnose the per-rank cost of the peer exchange (dev tool): for one shard
geometry, time sp_score, sp_score_peer with world = 1, and the rank-0 replay
of a world-P run (tools/peer_replay.py); with a -DSP_FUSED_TRACE build
(SP_LIB_AB=build/ab/trace.so) also print each launch's per-unit timeline
(MMA start period, statistics published -> lse2 ready).

  SP_LIB_AB=build/ab/trace.so python tools/peer_diag.py N P
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402

n_shard, P = int(sys.argv[1]), int(sys.argv[2])
w = gen.CONFIGS["C3"].with_(N=n_shard * P)
Q, K, T = spgen_cuda.make_inputs(w)
shards = [K[:, :, :, p * n_shard:(p + 1) * n_shard] for p in range(P)]
K0 = shards[0]
trace = os.environ.get("SP_LIB_AB", "").endswith("trace.so")


def timed(fn, pre=None, n=8):
    ms = []
    for _ in range(n):
        if pre:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.min(ms[2:]))


def timeline(fn, plan, pre=None):
    if not trace:
        return ""
    grid, upj = plan["grid"], plan["units_per_job"]
    buf = torch.zeros(grid * (upj + 1) * 8 + 8000, dtype=torch.int64, device="cuda")
    if pre:
        pre()
    sp.lib().sp_trace_enable(buf.data_ptr(), buf.numel())
    fn()
    torch.cuda.synchronize()
    sp.lib().sp_trace_enable(None, 0)
    tr = buf[:grid * (upj + 1) * 8].view(grid, upj + 1, 8)[:, :upj].cpu().numpy().astype(np.float64)
    t0 = tr[tr > 0].min()
    tr = np.where(tr > 0, (tr - t0) / 1000.0, np.nan)
    per = np.nanmedian(np.diff(tr[:, :, 1], axis=1))
    lat = np.nanmedian(tr[:, :, 5] - tr[:, :, 3])
    agg = np.nanmedian(tr[:, :, 6] - tr[:, :, 5])
    return f"  | span {np.nanmax(tr):.1f} us, MMA period/unit {per:.2f} us, publish->lse2 {lat:.2f} us, lse2->agg done {agg:.2f} us"


out = torch.empty((1, n_shard), dtype=torch.float32, device="cuda")
pl = sp.score_plan(Q, K0, w.Rv)
f = lambda: sp.score(Q, K0, R_valid=w.Rv, scale=w.scale, out=out, algo="fused")  # noqa: E731
print(f"sp_score N={n_shard}: {timed(f):.4f} ms plan {pl['token_groups']}x{pl['unit_groups']}" + timeline(f, pl))
ws1 = torch.zeros(sp.score_peer_workspace_bytes(Q, K0, 1, 0, w.Rv), dtype=torch.uint8, device="cuda")
f1 = lambda: sp.score_peer(Q, K0, 0, 1, [0], 0, w.Rv, w.scale, out=out, ws=ws1)  # noqa: E731
pl1 = sp.score_peer_plan(Q, K0, 1, 0, w.Rv)
print(f"score_peer world=1: {timed(f1):.4f} ms plan {pl1['token_groups']}x{pl1['unit_groups']}" + timeline(f1, pl1))

# rank-0 replay of a world-P run
sms = torch.cuda.get_device_properties(0).multi_processor_count
budget = sms // P
nb = sp.score_peer_buffer_bytes(Q, K0, P, 0, w.Rv)
bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(P)]
ptrs = [b.data_ptr() for b in bufs]
streams = [torch.cuda.Stream() for _ in range(P)]
wsv = [torch.zeros(sp.score_peer_workspace_bytes(Q, shards[p], P, budget, w.Rv), dtype=torch.uint8, device="cuda")
       for p in range(P)]
torch.cuda.synchronize()
for p in range(P):
    sp.score_peer(Q, shards[p], p, P, ptrs, budget, w.Rv, w.scale, stream=streams[p], ws=wsv[p])
torch.cuda.synchronize()
words = bufs[0].view(torch.int64)
half = words.numel() // 2
saved = words[:half].clone()
nz = (saved.view(-1, P, 32)[:, 1:] != 0).float().mean().item()
ws0 = torch.zeros(sp.score_peer_workspace_bytes(Q, K0, P, 0, w.Rv), dtype=torch.uint8, device="cuda")


def prefill():
    par = int(ws0.view(torch.int32)[0].item()) & 1
    words[par * half:(par + 1) * half].copy_(saved)
    words[(1 - par) * half:(2 - par) * half].zero_()
    torch.cuda.synchronize()


fP = lambda: sp.score_peer(Q, K0, 0, P, ptrs, 0, w.Rv, w.scale, out=out, ws=ws0)  # noqa: E731
plP = sp.score_peer_plan(Q, K0, P, 0, w.Rv)
print(f"replay rank 0 of world={P}: {timed(fP, prefill):.4f} ms plan {plP['token_groups']}x{plP['unit_groups']} "
      f"(peer words present: {nz:.3f})" + timeline(fP, plP, prefill))
sp.check_device_error()
