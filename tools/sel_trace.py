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


def read(reset=True):
    buf = (C.c_uint64 * 8)()
    assert lib.sp_select_trace_read(buf, 1 if reset else 0) == 0
    return list(buf)


def show(tag, t):
    t0 = t[1]
    names = ["entry", "past_wait", "A_done", "BC_start", "B_done", "C_done"]
    parts = "  ".join(f"{n}={(t[i] - t0) / 1e3:+.2f}" for i, n in enumerate(names))
    print(f"  {tag:12s} {parts} us", flush=True)


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
    for it in range(5):
        sp.select(imp, w.keep, w.pool_k, w.chunk, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)
        torch.cuda.synchronize()
        read(True)
        sp.select(imp, w.keep, w.pool_k, w.chunk, ids=ids, pos=pos, n_kept=nk, tokens=T, out=out)
        t = read(True)
        if it >= 2:
            show("alone", t)
    del Q, K, T
