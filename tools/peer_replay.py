"""Per-rank kernel time of the sequence-sharded single pass (sp_score_peer) for
one rank of a P-GPU run, measured on one GPU (dev tool).

The P ranks are first run once as co-scheduled virtual ranks (SMs/P CTAs each)
so that every rank word of every unit exists.  Rank 0's kernel is then
launched alone with the whole GPU (sm_budget 0, the plan a real rank uses),
with both halves of its rank-word buffer holding the other ranks' words (rank
0 never writes its own buffer's rows): each launch streams its 1/P shard and
merges the world rank words exactly as on a real rank, minus the wait for the
slowest peer.  20 back-to-back launches in a CUDA graph, timed with events.

  python tools/peer_replay.py C4 8 [C3 8 ...]      (C4 8:16,9 forces the plan n_tg,n_ug)
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


def replay(w, P, iters=5, plan_env=None):
    Q, K, T = spgen_cuda.make_inputs(w)
    n = w.N // P
    shards = [K[:, :, :, p * n:(p + 1) * n] for p in range(P)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    budget = sms // P
    nb = sp.score_peer_buffer_bytes(Q, shards[0], P, 0, w.Rv)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(P)]
    ptrs = [b.data_ptr() for b in bufs]
    # 1. every rank word exists: one co-scheduled virtual-rank call
    streams = [torch.cuda.Stream() for _ in range(P)]
    wsv = [torch.zeros(sp.score_peer_workspace_bytes(Q, shards[p], P, budget, w.Rv), dtype=torch.uint8,
                       device="cuda") for p in range(P)]
    torch.cuda.synchronize()
    for p in range(P):
        sp.score_peer(Q, shards[p], p, P, ptrs, budget, w.Rv, w.scale, stream=streams[p], ws=wsv[p])
    torch.cuda.synchronize()
    sp.check_device_error()
    words = bufs[0].view(torch.int64)
    half = words.numel() // 2
    saved = words[:half].clone()
    words[half:].copy_(saved)                         # both parity halves: the peers' words of every unit
    # 2. rank 0 alone on the whole GPU (optionally under a forced plan)
    if plan_env:
        os.environ["SP_FUSED_PLAN"] = plan_env
    ws0 = torch.zeros(sp.score_peer_workspace_bytes(Q, shards[0], P, 0, w.Rv), dtype=torch.uint8, device="cuda")
    out = torch.empty((w.B, n), dtype=torch.float32, device="cuda")
    plan = sp.score_peer_plan(Q, shards[0], P, 0, w.Rv)

    def run():
        sp.score_peer(Q, shards[0], 0, P, ptrs, 0, w.Rv, w.scale, out=out, ws=ws0)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            run()
    ms = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 20)
    sp.check_device_error()
    assert torch.equal(out, ref)
    os.environ.pop("SP_FUSED_PLAN", None)
    full = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")[:, :n]
    err = ((out - full).abs() / full.abs().clamp_min(1e-30)).max().item()
    return plan, ms, err, n


if __name__ == "__main__":
    args = sys.argv[1:]
    for i in range(0, len(args), 2):
        name, Ps = args[i], args[i + 1]
        P, plan_env = (int(Ps.split(":")[0]), Ps.split(":")[1]) if ":" in Ps else (int(Ps), None)
        w = gen.CONFIGS[name]
        plan, ms, err, n = replay(w, P, plan_env=plan_env)
        best = float(np.min(ms))
        kb = w.k_bytes / P
        print(f"{name} P={P}: rank-0 kernel {best:.4f} ms (min; median {np.median(ms):.4f}), "
              f"{kb / best / 1e6:.0f} GB/s of its {kb / 2**30:.2f} GiB shard, rel diff vs sp_score {err:.1e}; "
              f"plan n_tg {plan['token_groups']} n_ug {plan['unit_groups']} hier {plan['hier']} "
              f"tiles/job {plan['tiles_per_job']} grid {plan['grid']}", flush=True)
        torch.cuda.empty_cache()
