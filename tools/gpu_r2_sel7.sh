#!/bin/bash
# Timelines of the selection phases and of the score kernel's epilogue chunk phase (trace build), both libraries timed.
cd /root/repo; mkdir -p gpurun_out; exec > >(tee gpurun_out/sel7.log) 2>&1
SP_LIB_AB=build/ab/seltrace.so timeout 300 python tools/sel_trace.py
echo "--- product build"
SEL_CFGS=C3,C1 timeout 300 python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2502_02789_b200 as sp
from spgen import cuda as spgen_cuda
from spgen import gen
for cfg in ("C3", "C1"):
    w = gen.CONFIGS[cfg]
    Q, K, T = spgen_cuda.make_inputs(w)
    imp = torch.empty((w.B, w.N), dtype=torch.float32, device="cuda")
    cs = torch.empty((w.B, (w.N + w.chunk - 1) // w.chunk), dtype=torch.float32, device="cuda")
    for name, fn in [("score", lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=imp, algo="fused")),
                     ("score_chunks", lambda: sp.score_chunks(Q, K, w.pool_k, w.chunk, R_valid=w.Rv, scale=w.scale, out=imp, cs=cs)),
                     ("score", lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=imp, algo="fused"))]:
        for _ in range(3): fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): fn()
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        print(f"{cfg} graph-timed {name:13s} {a.elapsed_time(b) / 20 * 1e3:8.1f} us", flush=True)
    del Q, K, T
PY
