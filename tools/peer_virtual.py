"""Sequence-sharded single pass (sp_score_peer) as P virtual ranks on one GPU:
P co-scheduled launches on P streams, each capped at SMs/P CTAs, exchanging
statistics through each other's partial buffers (debug/validation tool)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402


def run(w, P, iters=3, check=None):
    Q, K, T = spgen_cuda.make_inputs(w)
    n = w.N // P
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    budget = sms // P
    shards = [K[:, :, :, p * n:(p + 1) * n] for p in range(P)]
    plan = sp.score_peer_plan(Q, shards[0], P, budget, w.Rv)
    nb = sp.score_peer_buffer_bytes(Q, shards[0], P, budget, w.Rv)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(P)]
    ptrs = [b.data_ptr() for b in bufs]
    streams = [torch.cuda.Stream() for _ in range(P)]
    outs = [torch.empty((w.B, n), dtype=torch.float32, device="cuda") for _ in range(P)]
    torch.cuda.synchronize()
    res, ms = [], []
    for _ in range(iters):
        t0 = time.perf_counter()
        for p in range(P):
            sp.score_peer(Q, shards[p], p, P, ptrs, budget, w.Rv, w.scale, out=outs[p], stream=streams[p])
        torch.cuda.synchronize()                      # the cross-rank barrier between calls
        ms.append((time.perf_counter() - t0) * 1e3)
        sp.check_device_error()
        res.append(torch.cat(outs, dim=1).clone())
    return plan, res, ms, (Q, K)


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = gen.CONFIGS[name]
    plan, res, ms, (Q, K) = run(w, P)
    full = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    err = (res[-1] - full).abs().div(full.abs().clamp_min(1e-30)).max().item()
    same = all(torch.equal(r, res[0]) for r in res)
    print(f"{name} P={P} plan={plan} max rel err vs sp_score {err:.2e} repeatable={same} wall ms {np.round(ms, 2)}")
