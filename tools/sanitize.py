"""Small invocations of every kernel family for compute-sanitizer runs (dev tool):
fused + SIMT score (C0, a C1-shaped 2K prompt), score_select (deferred finalize and
the epilogue chunk phase), select / select_gather /
ragged select, the sequence-sharded select (2 virtual ranks), paged and e4m3
score, the split API and the head-sharded accumulate."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import fp8, gen, paged  # noqa: E402

for w in (gen.CONFIGS["C0"], gen.CONFIGS["C1"].with_(N=2048, L=4)):
    Q, K, T = spgen_cuda.make_inputs(w)
    for algo in ("fused", "simt"):
        r = sp.specprefill(Q, K, T, w.keep, w.pool_k, w.chunk, scale=w.scale, algo=algo)
    imp = r["importance"]
    sp.select(imp, w.keep, w.pool_k, w.chunk, tokens=T)
    sp.select_ragged(imp, torch.full((w.B,), w.N // 2 + 1, dtype=torch.int32, device="cuda"), w.keep, w.pool_k,
                     w.chunk, tokens=T)
    if w.N % 2 == 0 and (w.N // 2) % w.chunk == 0:
        n = w.N // 2
        sh = [imp[:, :n].contiguous(), imp[:, n:].contiguous()]
        e = torch.stack([sp.seq_edges(x, 2, w.N, w.keep, w.pool_k, w.chunk) for x in sh]).contiguous()
        c = torch.stack([sp.seq_candidates(sh[p], e, p, 2, w.N, w.keep, w.pool_k, w.chunk) for p in range(2)])
        sp.seq_merge(c.contiguous(), 2, w.N, w.keep, w.pool_k, w.chunk, tokens=T)
    # sp_score_select: the deferred finalize (selection computes the importance) and
    # the epilogue chunk-phase variant (score kernel computes the chunk means)
    sp.score_select(Q, K, w.keep, w.pool_k, w.chunk, tokens=T, R_valid=w.Rv, scale=w.scale)
    os.environ["SP_SELECT_EPILOGUE"] = "1"
    sp.score_select(Q, K, w.keep, w.pool_k, w.chunk, tokens=T, R_valid=w.Rv, scale=w.scale)
    del os.environ["SP_SELECT_EPILOGUE"]
    st = sp.score_stats(Q, K, w.Rv, w.scale)
    lse2 = sp.stats_combine(st[None].contiguous())
    sp.score_finish(Q, K, lse2, w.Rv, w.scale)
    sp.acc_importance(sp.score_acc(Q, K, w.Rv, w.scale))
    cache, bt = paged.to_paged(K, 16)
    sp.score_paged(Q, cache, bt, N=w.N, scale=w.scale)
    if w.d % 32 == 0:                                  # (e4m3 rows are 32-byte multiples)
        q8, k8 = fp8.to_e4m3_codes(Q, fp8.Q_INV_SCALE), fp8.to_e4m3_codes(K, fp8.K_INV_SCALE)
        sp.score_e4m3(q8, k8, 1 / fp8.Q_INV_SCALE, 1 / fp8.K_INV_SCALE, scale=w.scale)
    torch.cuda.synchronize()
    sp.check_device_error()
print("sanitize workload done")
