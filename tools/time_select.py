"""Time sp_select (+fused gather) alone for a few shapes (debug tool)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp

for (B, N, chunk, pool) in [(1, 1024, 32, 5), (1, 4096, 32, 5), (1, 32768, 32, 5), (1, 131072, 32, 5),
                            (1, 32768, 1, 5), (1, 32768, 32, 1), (64, 1024, 32, 5), (1, 131072, 1, 1), (1, 8192, 1, 5)]:
    imp = torch.rand((B, N), device="cuda") + 1e-3
    tok = torch.randint(0, 1000, (B, N), dtype=torch.int32, device="cuda")
    ids = torch.empty_like(tok)
    pos, nk, out = torch.empty_like(tok), torch.empty((B,), dtype=torch.int32, device="cuda"), torch.empty_like(tok)
    for _ in range(3):
        sp.select(imp, 0.1, pool, chunk, ids=ids, pos=pos, n_kept=nk, tokens=tok, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()                       # 20 launches, no host overhead in the timing
    with torch.cuda.graph(g):
        for _ in range(20):
            sp.select(imp, 0.1, pool, chunk, ids=ids, pos=pos, n_kept=nk, tokens=tok, out=out)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"B={B} N={N} chunk={chunk} pool={pool}: {a.elapsed_time(b) / 20 * 1000:.1f} us")
