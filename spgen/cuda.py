"""ctypes loader of libspgen.so: device-side fill with the spgen generator
(bit-identical to spgen.gen).  Test/bench infrastructure, not product code."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import gen

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspgen.so")
_h = None


def _lib():
    global _h
    if _h is None:
        if not os.path.exists(_PATH):
            raise ImportError(f"{_PATH} missing; run __graft_entry__.build()")
        h = C.CDLL(_PATH)
        L, I, V, U = C.c_longlong, C.c_int, C.c_void_p, C.c_ulonglong
        h.spgen_fill_K.argtypes = [V, L, L, L, L, I, I, I, I, L, L, L, U, V, I, V, I, I, V]
        h.spgen_fill_Q.argtypes = [V, L, L, L, L, I, I, I, I, I, I, U, I, V]
        h.spgen_fill_tokens.argtypes = [V, I, L, U, V]
        h.spgen_read_stream.argtypes = [V, L, I, V, V]
        for f in (h.spgen_fill_K, h.spgen_fill_Q, h.spgen_fill_tokens, h.spgen_read_stream):
            f.restype = C.c_int
        _h = h
    return _h


def _stream():
    return torch.cuda.current_stream().cuda_stream


def spans_tensor(w: gen.Workload, device) -> torch.Tensor:
    sp = torch.full((w.B, 4, 2), -1, dtype=torch.int64)
    for b in range(w.B):
        for j, (s, e) in enumerate(gen.needle_spans(w, b)):
            sp[b, j, 0], sp[b, j, 1] = s, e
    return sp.to(device)


def fill_K(K: torch.Tensor, w: gen.Workload, i0: int = 0):
    """K: bf16 [B][L][Hkv][n_local][d] view (any strides, d contiguous) filled
    with global tokens [i0, i0 + n_local) of workload w."""
    B, L, Hkv, n, d = K.shape
    sp = spans_tensor(w, K.device)
    tiers = None
    if w.planted:
        tiers = torch.tensor(np.stack([gen.planted_tiers(w, b) for b in range(B)]).astype(np.int8), device=K.device)
    rc = _lib().spgen_fill_K(K.data_ptr(), K.stride(0), K.stride(1), K.stride(2), K.stride(3), B, L, Hkv, d,
                             w.N, i0, n, w.seed, sp.data_ptr(), int(w.values == "randn"),
                             None if tiers is None else tiers.data_ptr(), w.chunk, w.pool_k, _stream())
    if rc:
        raise RuntimeError(f"spgen_fill_K failed ({rc})")
    torch.cuda.current_stream().synchronize()        # keep `sp` / `tiers` alive until the kernel ran


def fill_Q(Q: torch.Tensor, w: gen.Workload):
    B, L, R, H, d = Q.shape
    rc = _lib().spgen_fill_Q(Q.data_ptr(), Q.stride(0), Q.stride(1), Q.stride(2), Q.stride(3), B, L, R, H, w.Hkv, d,
                             w.seed, int(w.values == "randn"), _stream())
    if rc:
        raise RuntimeError(f"spgen_fill_Q failed ({rc})")


def fill_tokens(tok: torch.Tensor, w: gen.Workload):
    B, N = tok.shape
    rc = _lib().spgen_fill_tokens(tok.data_ptr(), B, N, w.seed, _stream())
    if rc:
        raise RuntimeError(f"spgen_fill_tokens failed ({rc})")


def make_inputs(w: gen.Workload, device="cuda", i0: int = 0, n_local: int | None = None, k_pad: int = 0):
    """Device tensors (Q, K, tokens) of workload w; K holds tokens [i0, i0+n_local).
    k_pad > 0 allocates a larger cache (n_local + k_pad rows per head) and
    returns a strided view, to exercise non-contiguous layouts."""
    n = w.N - i0 if n_local is None else n_local
    Q = torch.empty((w.B, w.L, w.R, w.H, w.d), dtype=torch.bfloat16, device=device)
    Kbuf = torch.empty((w.B, w.L, w.Hkv, n + k_pad, w.d), dtype=torch.bfloat16, device=device)
    K = Kbuf[:, :, :, :n, :]
    tok = torch.empty((w.B, w.N), dtype=torch.int32, device=device)
    fill_Q(Q, w)
    fill_K(K, w, i0)
    fill_tokens(tok, w)
    return Q, K, tok


def read_stream_gbs(device, nbytes: int = 2 << 30, reps: int = 10) -> dict:
    """Measured HBM read-only streaming rate (bench's second roofline
    denominator): the best of `reps` passes over an nbytes buffer, for the TMA
    bulk-copy probe and the 128-bit load probe (spgen/probe.cu)."""
    buf = torch.ones(nbytes // 4, dtype=torch.int32, device=device)
    sink = torch.zeros(1, dtype=torch.int32, device=device)
    out = {}
    for mode, name in ((0, "tma_bulk"), (1, "ld_v4")):
        best = None
        for _ in range(reps + 2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = _lib().spgen_read_stream(buf.data_ptr(), nbytes, mode, sink.data_ptr(), _stream())
            b.record()
            b.synchronize()
            if rc:
                raise RuntimeError(f"spgen_read_stream failed ({rc})")
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        out[name] = nbytes / (best / 1000.0) / 1e9
    del buf
    return out
