"""Selection timeline (debug; needs a -DSP_SELECT_TRACE build:
tools/ab_build.sh WORKTREE seltrace -DSP_SELECT_TRACE, then SP_LIB_AB=build/ab/seltrace.so).
Prints, per config, the globaltimer stamps of the selection's phases after the
score kernel (score + select as in the bench step) and for select alone."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_02789_b200 as sp  # noqa: E402
from paper_2502_02789_b200 import _lib  # noqa: E402
from spgen import cuda as spgen_cuda  # noqa: E402
from spgen import gen  # noqa: E402

lib = C.CDLL(os.environ["SP_LIB_AB"])
lib.sp_select_trace_read.argtypes = [C.POINTER(C.c_uint64), C.c_int]


HAS_CHUNK = hasattr(lib, "sp_chunk_trace_read")
if HAS_CHUNK:
    lib.sp_chunk_trace_read.argtypes = [C.POINTER(C.c_uint64), C.c_int]


def read(reset=True):
    buf = (C.c_uint64 * 16)()
    assert lib.sp_select_trace_read(buf, 1 if reset else 0) == 0
    t = list(buf)
    ch = None
    if HAS_CHUNK:
        cb = (C.c_uint64 * 1280)()
        assert lib.sp_chunk_trace_read(cb, 1 if reset else 0) == 0
        ch = [list(cb[8 * i:8 * i + 8]) for i in range(160)]
    return t, ch


def show(tag, tc):
    t, ch = tc
    t0 = t[1]
    names = ["entry", "past_wait", "A_done", "BC_start", "B_done", "C_done", "A_staged", "A_pooled", "A_summed",
             "-", "pass0", "pass1", "pass2", "pass3"]
    parts = "  ".join(f"{n}={(t[i] - t0) / 1e3:+.2f}" for i, n in enumerate(names) if t[i] not in (0, 2**64 - 1)
                      and n != "-")
    print(f"  {tag:12s} {parts} us", flush=True)
    if ch is not None:
        rows = [r for r in ch if r[0] != 0]
        if rows:
            e0 = min(r[0] for r in rows)
            ends = sorted((max(r[:4]) - e0) / 1e3 for r in rows)
            own = [r for r in rows if r[1] != 0]
            def st(k, base=0):
                v = sorted((r[k] - (e0 if base is None else r[base])) / 1e3 for r in rows if r[k] and (base is None or r[base]))
                return f"med {v[len(v) // 2]:.2f} max {v[-1]:.2f}" if v else "-"
            print(f"     per CTA (us after its epilogue start): partials in {st(4)}, slice done {st(5)}, "
                  f"teardown start {st(6)}, exit {st(7)}; exit after first epilogue start {st(7, None)}; "
                  f"select past_wait after last exit {(t[1] - max(r[7] for r in rows if r[7])) / 1e3 if any(r[7] for r in rows) else 0:.2f}",
                  flush=True)
            wait = sorted((r[2] - r[1]) / 1e3 for r in own if r[2])
            dur = sorted((r[3] - r[2]) / 1e3 for r in own if r[3] and r[2])
            print(f"     score CTAs {len(rows)}: epilogue start spread {(max(r[0] for r in rows) - e0) / 1e3:.2f} us, "
                  f"CTA end (last stamp) median {ends[len(ends) // 2]:.2f} max {ends[-1]:.2f}; owners {len(own)}: "
                  f"wait median {wait[len(wait) // 2] if wait else 0:.2f} max {wait[-1] if wait else 0:.2f}, "
                  f"chunk work median {dur[len(dur) // 2] if dur else 0:.2f} max {dur[-1] if dur else 0:.2f}; "
                  f"score end -> select past_wait {(t[1] - e0) / 1e3 - ends[-1]:.2f} us", flush=True)


for cfg in os.environ.get("SEL_CFGS", "C3,C1").split(","):
    w = gen.CONFIGS[cfg]
    Q, K, T = spgen_cuda.make_inputs(w)
    imp = torch.empty((w.B, w.N), dtype=torch.float32, device="cuda")
    ids = torch.empty((w.B, w.N), dtype=torch.int32, device="cuda")
    pos, out = torch.empty_like(ids), torch.empty_like(ids)
    nk = torch.empty((w.B,), dtype=torch.int32, device="cuda")
    print(f"{cfg}: N={w.N} B={w.B} chunk={w.chunk} pool={w.pool_k} keep={w.keep}")
    for it in range(6):
        read(True)
        sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=imp, algo="fused")
        sp.select(imp, w.keep, w.pool_k, w.chunk, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)
        t = read(True)
        if it >= 3:
            show("after score", t)
    for it in range(6):
        read(True)
        sp.score_select(Q, K, w.keep, w.pool_k, w.chunk, w.pos0, tokens=T, R_valid=w.Rv, scale=w.scale,
                        out={"importance": imp, "ids": ids, "pos": pos, "n_kept": nk, "out_tokens": out})
        t = read(True)
        if it >= 3:
            show("score_select", t)
    for it in range(5):
        sp.select(imp, w.keep, w.pool_k, w.chunk, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)
        torch.cuda.synchronize()
        read(True)
        sp.select(imp, w.keep, w.pool_k, w.chunk, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)
        t = read(True)
        if it >= 2:
            show("alone", t)
    if os.environ.get("SEL_GTIME", "1") == "1":
        cs = torch.empty((w.B, (w.N + w.chunk - 1) // w.chunk), dtype=torch.float32, device="cuda")
        for name, fn in [("score", lambda: sp.score(Q, K, R_valid=w.Rv, scale=w.scale, out=imp, algo="fused")),
                         ("score_chunks", lambda: sp.score_chunks(Q, K, w.pool_k, w.chunk, R_valid=w.Rv,
                                                                  scale=w.scale, out=imp, cs=cs))]:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            print(f"  graph-timed {name:13s} {a.elapsed_time(b) / 20 * 1e3:8.1f} us", flush=True)
    del Q, K, T
