"""Thin PyTorch-facing wrappers over the C ABI (argument marshalling only).

PyTorch provides device memory and streams; every step of the path runs in the
CUDA kernels of libspecprefill.so.  Names follow the paper's Alg.1:
``score`` = compute_attention_score + aggregate_attention_score, ``select`` =
chunk_select_from_smoothed_attention + restore_pos_ids, ``gather`` = the
token gather of merge_requests.

Tensor layouts (strides are passed through, the head dim must be contiguous):
  Q  bf16 [B][L][R][H][d]     look-ahead query rows (post-RoPE)
  K  bf16 [B][L][Hkv][N][d]   speculator key cache
"""
from __future__ import annotations

import collections
import ctypes as C
import math

import torch

from . import _lib
from ._lib import check, lib

ALGOS = {"auto": _lib.SP_SCORE_AUTO, "fused": _lib.SP_SCORE_FUSED, "simt": _lib.SP_SCORE_SIMT}

_ws_cache: "collections.OrderedDict" = collections.OrderedDict()
_WS_MAX = 64


def _stream_ptr(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def workspace(tag, nbytes: int, device, stream=None) -> torch.Tensor:
    """Zero-initialised, cached device workspace, one per (tag, device, stream).
    The fused kernel leaves its counters at zero after every call, but their
    position depends on the geometry, so a workspace is only ever reused for
    the same ``tag`` (which includes the geometry) and the same stream (two
    streams never share a launch epoch or partial buffers): see
    include/specprefill.h, "Ownership".  Least-recently-used entries beyond 64
    are dropped; a buffer used on a non-current stream is recorded on it, so
    the caching allocator does not hand its memory out while a kernel on that
    stream may still use it."""
    dev = torch.device(device)
    key = (tag, dev.index, _stream_ptr(stream))
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        while len(_ws_cache) >= _WS_MAX:
            _ws_cache.popitem(last=False)
        buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    else:
        _ws_cache.move_to_end(key)
    if stream is not None and stream != torch.cuda.current_stream(dev):
        buf.record_stream(stream)
    return buf


def _geom_key(g) -> tuple:
    """Workspace cache key: the geometry and the fused plan it runs with (the
    partial-statistics layout depends on the plan: env override, sp_score_tune)."""
    import os
    out = (C.c_int64 * _lib.PLAN_INFO)()
    plan = (out[2], out[3], out[9]) if lib().sp_score_plan(C.byref(g), out) == _lib.SP_OK else None
    return (g.B, g.L, g.H, g.Hkv, g.d, g.R, g.R_valid, g.N, os.environ.get("SP_FUSED_PLAN"), plan)


_E4M3 = (torch.float8_e4m3fn, torch.uint8)


def make_geom(Q: torch.Tensor, K: torch.Tensor, R_valid: int | None = None, scale: float | None = None,
              e4m3: bool = False):
    if e4m3:
        if Q.dtype not in _E4M3 or K.dtype not in _E4M3:
            raise TypeError("Q and K must be float8_e4m3fn (or uint8 holding e4m3 codes)")
    elif Q.dtype != torch.bfloat16 or K.dtype != torch.bfloat16:
        raise TypeError("Q and K must be bfloat16")
    if Q.dim() != 5 or K.dim() != 5:
        raise ValueError("Q must be [B][L][R][H][d] and K [B][L][Hkv][N][d]")
    B, L, R, H, d = Q.shape
    Bk, Lk, Hkv, N, dk = K.shape
    if (B, L, d) != (Bk, Lk, dk):
        raise ValueError(f"Q {tuple(Q.shape)} and K {tuple(K.shape)} disagree")
    if Q.stride(-1) != 1 or K.stride(-1) != 1:
        raise ValueError("head dim must be contiguous")
    g = _lib.sp_geom(B=B, L=L, H=H, Hkv=Hkv, d=d, R=R, R_valid=R if R_valid is None else R_valid, N=N,
                     scale=float(1.0 / math.sqrt(d)) if scale is None else float(scale))
    lay = _lib.sp_layout(k_b=K.stride(0), k_l=K.stride(1), k_g=K.stride(2), k_i=K.stride(3),
                         q_b=Q.stride(0), q_l=Q.stride(1), q_r=Q.stride(2), q_h=Q.stride(3))
    return g, lay


def score(Q, K, R_valid=None, scale=None, out=None, algo: str = "auto", stream=None) -> torch.Tensor:
    """Token importance [B][N] fp32 (O1-O4)."""
    g, lay = make_geom(Q, K, R_valid, scale)
    if out is None:
        out = torch.empty((g.B, g.N), dtype=torch.float32, device=K.device)
    a = ALGOS[algo]
    nbytes = lib().sp_score_workspace_bytes(C.byref(g), a)
    ws = workspace(("score", algo, _geom_key(g)), nbytes, K.device, stream)
    check(lib().sp_score_ex(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), out.data_ptr(), ws.data_ptr(),
                            ws.numel(), a, _stream_ptr(stream)), "sp_score")
    return out


def score_e4m3(Q8, K8, q_scale: float = 1.0, k_scale: float = 1.0, R_valid=None, scale=None, out=None,
               stream=None) -> torch.Tensor:
    """Row f4: token importance [B][N] fp32 from FP8 e4m3 Q/K codes with
    per-tensor dequantisation scales (Q = q_scale*Q8, K = k_scale*K8)."""
    g, lay = make_geom(Q8, K8, R_valid, scale, e4m3=True)
    if out is None:
        out = torch.empty((g.B, g.N), dtype=torch.float32, device=K8.device)
    nbytes = lib().sp_score_e4m3_workspace_bytes(C.byref(g))
    if nbytes == 0:
        check(_lib.SP_EUNSUPPORTED, "sp_score_e4m3")
    pl = (C.c_int64 * _lib.PLAN_INFO)()
    lib().sp_score_e4m3_plan(C.byref(g), pl)
    ws = workspace(("score_e4m3", _geom_key(g), (pl[2], pl[3], pl[9])), nbytes, K8.device, stream)
    check(lib().sp_score_e4m3(Q8.data_ptr(), K8.data_ptr(), float(q_scale), float(k_scale), C.byref(g), C.byref(lay),
                              out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_score_e4m3")
    return out


def score_e4m3_plan(Q8, K8, R_valid=None) -> dict:
    g, _ = make_geom(Q8, K8, R_valid, e4m3=True)
    out = (C.c_int64 * _lib.PLAN_INFO)()
    check(lib().sp_score_e4m3_plan(C.byref(g), out), "sp_score_e4m3_plan")
    return dict(zip(_lib.PLAN_KEYS, list(out)))


def score_lookahead(Q, K, K_la, la_shift: int = 0, R_valid=None, scale=None, out=None, stream=None) -> torch.Tensor:
    """Row f4, reading Z2': importance [B][N] with the look-ahead tokens' keys
    K_la (bf16 [B][L][Hkv][R][d], d contiguous) in each row's softmax denominator."""
    g, lay = make_geom(Q, K, R_valid, scale)
    if K_la.dtype != torch.bfloat16 or K_la.dim() != 5 or K_la.stride(-1) != 1:
        raise ValueError("K_la must be bf16 [B][L][Hkv][R][d] with d contiguous")
    la = _lib.sp_lookahead_k(K_la=K_la.data_ptr(), s_b=K_la.stride(0), s_l=K_la.stride(1), s_g=K_la.stride(2),
                             s_j=K_la.stride(3), la_shift=int(la_shift))
    if out is None:
        out = torch.empty((g.B, g.N), dtype=torch.float32, device=K.device)
    nbytes = lib().sp_score_lookahead_workspace_bytes(C.byref(g))
    if nbytes == 0:
        check(_lib.SP_EUNSUPPORTED, "sp_score_lookahead")
    ws = workspace(("score_la", _geom_key(g)), nbytes, K.device, stream)
    check(lib().sp_score_lookahead(Q.data_ptr(), K.data_ptr(), C.byref(la), C.byref(g), C.byref(lay), out.data_ptr(),
                                   ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_score_lookahead")
    return out


def score_paged(Q, K_cache, block_table, seq_lens=None, N=None, R_valid=None, scale=None, out=None,
                stream=None, q_scale=None, k_scale=None) -> torch.Tensor:
    """Row f3: token importance [B][N] fp32 from a paged K cache.

    K_cache: bf16 (or, with q_scale/k_scale, e4m3 codes) [L][num_blocks][block_size][Hkv][d],
    any strides with d contiguous (vLLM NHD storage, or an HND store viewed this way);
    block_table: int32 [B][max_blocks] (device); seq_lens: int32 [B] (device) or None;
    N: the longest prompt, the row length of the output (default max_blocks * block_size).
    Entries i >= seq_lens[b] of the output rows are left untouched."""
    e4m3 = q_scale is not None
    if e4m3:
        if Q.dtype not in _E4M3 or K_cache.dtype not in _E4M3:
            raise TypeError("with q_scale/k_scale, Q and K_cache must hold e4m3 codes")
    elif Q.dtype != torch.bfloat16 or K_cache.dtype != torch.bfloat16:
        raise TypeError("Q and K_cache must be bfloat16")
    if K_cache.dim() != 5 or Q.dim() != 5 or K_cache.stride(-1) != 1 or Q.stride(-1) != 1:
        raise ValueError("Q [B][L][R][H][d], K_cache [L][num_blocks][block_size][Hkv][d], d contiguous")
    if block_table.dtype != torch.int32 or not block_table.is_contiguous() or block_table.dim() != 2:
        raise ValueError("block_table must be contiguous int32 [B][max_blocks]")
    B, L, R, H, d = Q.shape
    Lk, nblk, bs, Hkv, dk = K_cache.shape
    if (Lk, dk) != (L, d) or block_table.shape[0] != B:
        raise ValueError("Q / K_cache / block_table disagree")
    N = block_table.shape[1] * bs if N is None else int(N)
    g = _lib.sp_geom(B=B, L=L, H=H, Hkv=Hkv, d=d, R=R, R_valid=R if R_valid is None else R_valid, N=N,
                     scale=float(1.0 / math.sqrt(d)) if scale is None else float(scale))
    lay = _lib.sp_layout(k_b=0, k_l=0, k_g=0, k_i=0, q_b=Q.stride(0), q_l=Q.stride(1), q_r=Q.stride(2),
                         q_h=Q.stride(3))
    if seq_lens is not None and (seq_lens.dtype != torch.int32 or not seq_lens.is_contiguous()):
        raise ValueError("seq_lens must be contiguous int32 [B]")
    pk = _lib.sp_paged_k(cache=K_cache.data_ptr(), s_l=K_cache.stride(0), s_blk=K_cache.stride(1),
                         s_tok=K_cache.stride(2), s_g=K_cache.stride(3), num_blocks=nblk, block_size=bs,
                         block_table=block_table.data_ptr(), max_blocks=block_table.shape[1],
                         seq_lens=None if seq_lens is None else seq_lens.data_ptr())
    if out is None:
        out = torch.zeros((B, N), dtype=torch.float32, device=K_cache.device)
    if e4m3:
        nbytes = lib().sp_score_e4m3_workspace_bytes(C.byref(g))
        if nbytes == 0:
            check(_lib.SP_EUNSUPPORTED, "sp_score_paged_e4m3")
        pl = (C.c_int64 * _lib.PLAN_INFO)()
        lib().sp_score_e4m3_plan(C.byref(g), pl)
        ws = workspace(("score_paged_e4m3", _geom_key(g), (pl[2], pl[3], pl[9])), nbytes, K_cache.device, stream)
        check(lib().sp_score_paged_e4m3(Q.data_ptr(), C.byref(pk), float(q_scale), float(k_scale), C.byref(g),
                                        C.byref(lay), out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
              "sp_score_paged_e4m3")
        return out
    nbytes = lib().sp_score_paged_workspace_bytes(C.byref(g))
    if nbytes == 0:
        check(_lib.SP_EUNSUPPORTED, "sp_score_paged")
    ws = workspace(("score_paged", _geom_key(g)), nbytes, K_cache.device, stream)
    check(lib().sp_score_paged(Q.data_ptr(), C.byref(pk), C.byref(g), C.byref(lay), out.data_ptr(), ws.data_ptr(),
                               ws.numel(), _stream_ptr(stream)), "sp_score_paged")
    return out


def select_ragged(importance: torch.Tensor, seq_lens: torch.Tensor, keep: float, pool_k: int, chunk: int,
                  pos0: int = 0, tokens=None, stream=None):
    """Row f3: per-request selection over importance[b][:seq_lens[b]];
    returns (ids, pos, n_kept) or (ids, pos, n_kept, gathered tokens)."""
    if importance.dtype != torch.float32 or importance.dim() != 2 or not importance.is_contiguous():
        raise ValueError("importance must be contiguous fp32 [B][N]")
    if seq_lens.dtype != torch.int32 or not seq_lens.is_contiguous():
        raise ValueError("seq_lens must be contiguous int32 [B]")
    B, N = importance.shape
    dev = importance.device
    p = _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))
    ids = torch.empty((B, N), dtype=torch.int32, device=dev)
    pos = torch.empty_like(ids)
    n_kept = torch.empty((B,), dtype=torch.int32, device=dev)
    out = torch.empty_like(ids) if tokens is not None else None
    nbytes = lib().sp_select_workspace_bytes(B, N, C.byref(p))
    if nbytes == 0:
        check(_lib.SP_EINVAL, "sp_select_ragged")
    ws = workspace(("select", B, N, int(chunk)), nbytes, dev, stream)
    check(lib().sp_select_ragged(importance.data_ptr(), seq_lens.data_ptr(),
                                 None if tokens is None else tokens.data_ptr(), B, N, C.byref(p), ids.data_ptr(),
                                 pos.data_ptr(), n_kept.data_ptr(), None if out is None else out.data_ptr(),
                                 ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_select_ragged")
    return (ids, pos, n_kept) if tokens is None else (ids, pos, n_kept, out)


def select(importance: torch.Tensor, keep: float, pool_k: int, chunk: int, pos0: int = 0, ids=None, pos=None,
           n_kept=None, stream=None, tokens=None, out=None):
    """(ids [B][N] int32, pos [B][N] int32, n_kept [B] int32); only the first
    n_kept[b] entries of row b are meaningful (O5-O9).  With
    ``tokens`` the gather is fused into the same launch and the gathered
    tokens are returned as a fourth element."""
    if importance.dtype != torch.float32 or importance.dim() != 2 or not importance.is_contiguous():
        raise ValueError("importance must be contiguous fp32 [B][N]")
    B, N = importance.shape
    dev = importance.device
    p = _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))
    ids = torch.empty((B, N), dtype=torch.int32, device=dev) if ids is None else ids
    pos = torch.empty((B, N), dtype=torch.int32, device=dev) if pos is None else pos
    n_kept = torch.empty((B,), dtype=torch.int32, device=dev) if n_kept is None else n_kept
    nbytes = lib().sp_select_workspace_bytes(B, N, C.byref(p))
    if nbytes == 0:
        check(_lib.SP_EINVAL, "sp_select")
    ws = workspace(("select", B, N, int(chunk)), nbytes, dev, stream)
    if tokens is None:
        check(lib().sp_select(importance.data_ptr(), B, N, C.byref(p), ids.data_ptr(), pos.data_ptr(),
                              n_kept.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_select")
        return ids, pos, n_kept
    if tokens.dtype != torch.int32 or not tokens.is_contiguous() or tuple(tokens.shape) != (B, N):
        raise ValueError("tokens must be contiguous int32 [B][N]")
    out = torch.empty_like(tokens) if out is None else out
    check(lib().sp_select_gather(importance.data_ptr(), tokens.data_ptr(), B, N, C.byref(p), ids.data_ptr(),
                                 pos.data_ptr(), n_kept.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                 _stream_ptr(stream)), "sp_select_gather")
    return ids, pos, n_kept, out


def _seq_params(keep, pool_k, chunk, pos0=0):
    return _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))


def seq_candidate_count(N: int, world: int, keep: float, pool_k: int, chunk: int) -> int:
    """M = min(K_c, n_c / world): candidates per rank of the sequence-sharded select."""
    p = _seq_params(keep, pool_k, chunk)
    m = lib().sp_seq_candidate_count(int(N), int(world), C.byref(p))
    if m < 0:
        check(_lib.SP_EINVAL, "sp_seq_candidate_count")
    return int(m)


def seq_edges(imp_local: torch.Tensor, world: int, N: int, keep: float, pool_k: int, chunk: int,
              stream=None) -> torch.Tensor:
    """Sequence-sharded select, step 1: this rank's first and last (pool_k-1)/2
    importance values, edges [B][2w] fp32 (all-gathered by the caller)."""
    if imp_local.dtype != torch.float32 or imp_local.dim() != 2 or not imp_local.is_contiguous():
        raise ValueError("imp_local must be contiguous fp32 [B][N/world]")
    B = imp_local.shape[0]
    w = (int(pool_k) - 1) // 2
    edges = torch.empty((B, 2 * w), dtype=torch.float32, device=imp_local.device)
    p = _seq_params(keep, pool_k, chunk)
    check(lib().sp_seq_edges(imp_local.data_ptr(), B, int(N), int(world), C.byref(p),
                             edges.data_ptr() if w else None, _stream_ptr(stream)), "sp_seq_edges")
    return edges


def seq_candidates(imp_local: torch.Tensor, edges_all, rank: int, world: int, N: int, keep: float, pool_k: int,
                   chunk: int, stream=None) -> torch.Tensor:
    """Step 3: pool + chunk means of this rank's chunks and its top-M
    candidates, int64 [B][M] keys (fp32 score bits << 32 | ~global chunk id;
    unsigned order = (score desc, index asc)), in chunk order."""
    if imp_local.dtype != torch.float32 or imp_local.dim() != 2 or not imp_local.is_contiguous():
        raise ValueError("imp_local must be contiguous fp32 [B][N/world]")
    B = imp_local.shape[0]
    p = _seq_params(keep, pool_k, chunk)
    M = seq_candidate_count(N, world, keep, pool_k, chunk)
    cand = torch.empty((B, M), dtype=torch.int64, device=imp_local.device)
    nbytes = lib().sp_seq_select_workspace_bytes(B, int(N), int(world), C.byref(p))
    if nbytes == 0:
        check(_lib.SP_EINVAL, "sp_seq_candidates")
    ws = workspace(("seq_sel", B, int(N), int(world), int(chunk)), nbytes, imp_local.device, stream)
    if edges_all is not None and (edges_all.dtype != torch.float32 or not edges_all.is_contiguous()):
        raise ValueError("edges_all must be contiguous fp32 [world][B][2w]")
    check(lib().sp_seq_candidates(imp_local.data_ptr(), None if edges_all is None or edges_all.numel() == 0
                                  else edges_all.data_ptr(), int(rank), int(world), B, int(N), C.byref(p),
                                  cand.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
          "sp_seq_candidates")
    return cand


def seq_merge(cand_all: torch.Tensor, world: int, N: int, keep: float, pool_k: int, chunk: int, pos0: int = 0,
              tokens=None, stream=None):
    """Step 5: global top-K_c of the gathered candidates [world][B][M] ->
    (ids, pos, n_kept[, gathered tokens]) for the whole prompt, as select()."""
    if cand_all.dtype != torch.int64 or cand_all.dim() != 3 or not cand_all.is_contiguous():
        raise ValueError("cand_all must be contiguous int64 [world][B][M]")
    B = cand_all.shape[1]
    dev = cand_all.device
    p = _seq_params(keep, pool_k, chunk, pos0)
    ids = torch.empty((B, N), dtype=torch.int32, device=dev)
    pos = torch.empty_like(ids)
    n_kept = torch.empty((B,), dtype=torch.int32, device=dev)
    out = None
    if tokens is not None:
        if tokens.dtype != torch.int32 or not tokens.is_contiguous() or tuple(tokens.shape) != (B, N):
            raise ValueError("tokens must be contiguous int32 [B][N]")
        out = torch.empty_like(tokens)
    nbytes = lib().sp_seq_select_workspace_bytes(B, int(N), int(world), C.byref(p))
    if nbytes == 0:
        check(_lib.SP_EINVAL, "sp_seq_merge")
    ws = workspace(("seq_sel", B, int(N), int(world), int(chunk)), nbytes, dev, stream)
    check(lib().sp_seq_merge(cand_all.data_ptr(), int(world), B, int(N), C.byref(p),
                             None if tokens is None else tokens.data_ptr(), ids.data_ptr(), pos.data_ptr(),
                             n_kept.data_ptr(), None if out is None else out.data_ptr(), ws.data_ptr(), ws.numel(),
                             _stream_ptr(stream)), "sp_seq_merge")
    return (ids, pos, n_kept) if tokens is None else (ids, pos, n_kept, out)


def score_select(Q, K, keep: float, pool_k: int, chunk: int, pos0: int = 0, tokens=None, R_valid=None, scale=None,
                 out=None, stream=None):
    """sp_score + sp_select_gather in one call: the fused score kernel computes the
    selection's chunk scores in its epilogue and the dependent selection launch
    runs the top-K_c and the compaction (same bits as the two calls).
    Returns (importance, ids, pos, n_kept[, gathered tokens]); ``out`` may hold
    preallocated tensors with those keys."""
    g, lay = make_geom(Q, K, R_valid, scale)
    p = _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))
    dev = K.device
    o = dict(out or {})
    imp = o.get("importance") if o.get("importance") is not None else torch.empty((g.B, g.N), dtype=torch.float32,
                                                                                  device=dev)
    ids = o.get("ids") if o.get("ids") is not None else torch.empty((g.B, g.N), dtype=torch.int32, device=dev)
    pos = o.get("pos") if o.get("pos") is not None else torch.empty((g.B, g.N), dtype=torch.int32, device=dev)
    nk = o.get("n_kept") if o.get("n_kept") is not None else torch.empty((g.B,), dtype=torch.int32, device=dev)
    outt = None
    if tokens is not None:
        if tokens.dtype != torch.int32 or not tokens.is_contiguous() or tuple(tokens.shape) != (g.B, g.N):
            raise ValueError("tokens must be contiguous int32 [B][N]")
        outt = o.get("out_tokens") if o.get("out_tokens") is not None else torch.empty_like(tokens)
    nbytes = lib().sp_score_select_workspace_bytes(C.byref(g), C.byref(p))
    if nbytes == 0:
        check(_lib.SP_EINVAL, "sp_score_select")
    ws = workspace(("score_select", _geom_key(g), int(chunk), int(pool_k), float(keep)), nbytes, dev, stream)
    check(lib().sp_score_select(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), C.byref(p),
                                None if tokens is None else tokens.data_ptr(), imp.data_ptr(), ids.data_ptr(),
                                pos.data_ptr(), nk.data_ptr(), None if outt is None else outt.data_ptr(),
                                ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_score_select")
    return (imp, ids, pos, nk) if tokens is None else (imp, ids, pos, nk, outt)


def score_chunks(Q, K, pool_k: int, chunk: int, R_valid=None, scale=None, out=None, cs=None, stream=None):
    """The score kernel of score_select alone: (importance [B][N], chunk scores
    [B][ceil(N / chunk)]) -- the selection's pooled chunk means computed in the
    kernel's epilogue (same bits as the selection's own).  Raises SpError
    (unsupported) where the plan cannot stage them."""
    g, lay = make_geom(Q, K, R_valid, scale)
    dev = K.device
    n_c = (g.N + int(chunk) - 1) // int(chunk)
    out = torch.empty((g.B, g.N), dtype=torch.float32, device=dev) if out is None else out
    cs = torch.empty((g.B, n_c), dtype=torch.float32, device=dev) if cs is None else cs
    nbytes = lib().sp_score_workspace_bytes(C.byref(g), ALGOS["fused"])
    ws = workspace(("score", "fused", _geom_key(g)), nbytes, dev, stream)
    check(lib().sp_score_chunks(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), int(pool_k), int(chunk),
                                out.data_ptr(), cs.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
          "sp_score_chunks")
    return out, cs


def gather(tokens: torch.Tensor, ids: torch.Tensor, n_kept: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """out[b][j] = tokens[b][ids[b][j]] for j < n_kept[b] (bit-exact)."""
    if tokens.dtype != torch.int32 or not tokens.is_contiguous():
        raise ValueError("tokens must be contiguous int32 [B][N]")
    B, N = tokens.shape
    out = torch.empty_like(tokens) if out is None else out
    check(lib().sp_gather(tokens.data_ptr(), ids.data_ptr(), n_kept.data_ptr(), B, N, out.data_ptr(),
                          _stream_ptr(stream)), "sp_gather")
    return out


def score_tune(Q, K, R_valid=None, scale=None, stream=None) -> dict:
    """Time the fused kernel's best plan candidates on these inputs and register
    the fastest for this geometry (sp_score_tune; synchronises, allocates)."""
    g, lay = make_geom(Q, K, R_valid, scale)
    out = (C.c_int64 * 3)()
    ms = C.c_float()
    check(lib().sp_score_tune(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), out, C.byref(ms),
                              _stream_ptr(stream)), "sp_score_tune")
    return {"token_groups": out[0], "unit_groups": out[1], "hier": out[2], "ms_per_launch": ms.value}


def score_e4m3_tune(Q8, K8, q_scale: float = 1.0, k_scale: float = 1.0, R_valid=None, scale=None,
                    stream=None) -> dict:
    g, lay = make_geom(Q8, K8, R_valid, scale, e4m3=True)
    out = (C.c_int64 * 3)()
    ms = C.c_float()
    check(lib().sp_score_e4m3_tune(Q8.data_ptr(), K8.data_ptr(), float(q_scale), float(k_scale), C.byref(g),
                                   C.byref(lay), out, C.byref(ms), _stream_ptr(stream)), "sp_score_e4m3_tune")
    return {"token_groups": out[0], "unit_groups": out[1], "hier": out[2], "ms_per_launch": ms.value}


def score_plan(Q, K, R_valid=None) -> dict:
    """The fused kernel's launch plan for this geometry on the current device."""
    g, _ = make_geom(Q, K, R_valid)
    out = (C.c_int64 * _lib.PLAN_INFO)()
    check(lib().sp_score_plan(C.byref(g), out), "sp_score_plan")
    return dict(zip(_lib.PLAN_KEYS, list(out)))


def score_stats(Q, K, R_valid=None, scale=None, out=None, stream=None) -> torch.Tensor:
    """Sequence-sharded split, step 1: local softmax statistics (log2 domain)
    stats [B*L*H*R_valid][2] = (m2, l) over this shard's tokens."""
    g, lay = make_geom(Q, K, R_valid, scale)
    rows = g.B * g.L * g.H * g.R_valid
    out = torch.empty((rows, 2), dtype=torch.float32, device=K.device) if out is None else out
    nbytes = lib().sp_score_split_workspace_bytes(C.byref(g))
    ws = workspace(("split", _geom_key(g), _split_algo()), nbytes, K.device, stream)
    check(lib().sp_score_stats(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), out.data_ptr(), ws.data_ptr(),
                               ws.numel(), _stream_ptr(stream)), "sp_score_stats")
    return out


def stats_combine(parts: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """Step 2: merge [P][rows][2] gathered statistics in rank order -> lse2 [rows]."""
    if parts.dtype != torch.float32 or parts.dim() != 3 or parts.shape[2] != 2 or not parts.is_contiguous():
        raise ValueError("parts must be contiguous fp32 [P][rows][2]")
    P, rows = parts.shape[0], parts.shape[1]
    out = torch.empty((rows,), dtype=torch.float32, device=parts.device) if out is None else out
    check(lib().sp_stats_combine(parts.data_ptr(), P, rows, out.data_ptr(), _stream_ptr(stream)), "sp_stats_combine")
    return out


def score_finish(Q, K, lse2, R_valid=None, scale=None, out=None, stream=None) -> torch.Tensor:
    """Step 3: importance over this shard's tokens given the global lse2."""
    g, lay = make_geom(Q, K, R_valid, scale)
    out = torch.empty((g.B, g.N), dtype=torch.float32, device=K.device) if out is None else out
    nbytes = lib().sp_score_split_workspace_bytes(C.byref(g))
    ws = workspace(("split", _geom_key(g), _split_algo()), nbytes, K.device, stream)
    check(lib().sp_score_finish(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), lse2.data_ptr(), out.data_ptr(),
                                ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_score_finish")
    return out


def score_acc(Q, K, R_valid=None, scale=None, out=None, stream=None) -> torch.Tensor:
    """Head-sharded partition (row f1): acc2 [B][R_valid][N] = max over this
    rank's (layer, head) of the log2-domain log-probability; MAX-reduce across
    ranks, then acc_importance."""
    g, lay = make_geom(Q, K, R_valid, scale)
    out = torch.empty((g.B, g.R_valid, g.N), dtype=torch.float32, device=K.device) if out is None else out
    nbytes = lib().sp_score_workspace_bytes(C.byref(g), _lib.SP_SCORE_FUSED)
    ws = workspace(("score", "fused", _geom_key(g)), nbytes, K.device, stream)
    check(lib().sp_score_acc(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), out.data_ptr(), ws.data_ptr(),
                             ws.numel(), _stream_ptr(stream)), "sp_score_acc")
    return out


def acc_importance(acc2, out=None, stream=None) -> torch.Tensor:
    """importance[b][i] = mean_r 2^acc2[b][r][i] (after the cross-rank MAX)."""
    if acc2.dtype != torch.float32 or not acc2.is_contiguous() or acc2.dim() != 3:
        raise ValueError("acc2 must be contiguous fp32 [B][R_valid][N]")
    B, Rv, N = acc2.shape
    out = torch.empty((B, N), dtype=torch.float32, device=acc2.device) if out is None else out
    check(lib().sp_acc_importance(acc2.data_ptr(), B, Rv, N, out.data_ptr(), _stream_ptr(stream)),
          "sp_acc_importance")
    return out


def score_peer_buffer_bytes(Q, K, world: int, sm_budget: int = 0, R_valid=None) -> int:
    """Bytes of one rank's partial buffer for score_peer (this rank's shard geometry)."""
    g, _ = make_geom(Q, K, R_valid)
    return int(lib().sp_score_peer_buffer_bytes(C.byref(g), world, sm_budget))


def score_peer_plan(Q, K, world: int, sm_budget: int = 0, R_valid=None) -> dict:
    g, _ = make_geom(Q, K, R_valid)
    out = (C.c_int64 * _lib.PLAN_INFO)()
    check(lib().sp_score_peer_plan(C.byref(g), int(world), sm_budget, out), "sp_score_peer_plan")
    return dict(zip(_lib.PLAN_KEYS, list(out)))


def score_peer_workspace_bytes(Q, K, world: int, sm_budget: int = 0, R_valid=None) -> int:
    g, _ = make_geom(Q, K, R_valid)
    return int(lib().sp_score_peer_workspace_bytes(C.byref(g), int(world), sm_budget))


def score_peer(Q, K, rank: int, world: int, peer_ptrs, sm_budget: int = 0, R_valid=None, scale=None, out=None,
               stream=None, ws_tag=None, ws=None) -> torch.Tensor:
    """Sequence-sharded single pass: importance of this rank's tokens, the
    statistics exchanged in-kernel through the peers' partial buffers
    (peer_ptrs: `world` device addresses, rank order).  ``ws``: a zeroed
    workspace owned together with the peer buffers (its launch epoch selects
    the half of the peer buffers a launch writes, so the two must live and die
    together); by default one from the cache."""
    g, lay = make_geom(Q, K, R_valid, scale)
    out = torch.empty((g.B, g.N), dtype=torch.float32, device=K.device) if out is None else out
    nbytes = lib().sp_score_peer_workspace_bytes(C.byref(g), int(world), sm_budget)
    if nbytes == 0:
        check(_lib.SP_EUNSUPPORTED, "sp_score_peer")
    if ws is None:
        ws = workspace(("peer", _geom_key(g), world, sm_budget, rank if ws_tag is None else ws_tag), nbytes, K.device,
                       stream)
    elif ws.numel() < nbytes:
        raise ValueError("peer workspace too small")
    ptrs = (C.c_void_p * world)(*[int(x) for x in peer_ptrs])
    check(lib().sp_score_peer(Q.data_ptr(), K.data_ptr(), C.byref(g), C.byref(lay), rank, world, ptrs, sm_budget,
                              out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "sp_score_peer")
    return out


def _split_algo():
    import os
    return os.environ.get("SP_SPLIT_ALGO", "auto")


def kept_chunks(n_chunks: int, keep: float) -> int:
    k = lib().sp_kept_chunks(int(n_chunks), float(keep))
    if k < 0:
        raise ValueError("invalid keep rate / chunk count")
    return k


def check_device_error(stream=None):
    check(lib().sp_check_device_error(_stream_ptr(stream)), "device")


def specprefill(Q, K, tokens, keep, pool_k, chunk, R_valid=None, scale=None, pos0=0, algo="auto", stream=None):
    """The whole hot path (Alg.1): importance, kept ids, positions,
    gathered tokens, and the first decode position N + pos0."""
    imp = score(Q, K, R_valid, scale, algo=algo, stream=stream)
    ids, pos, n_kept = select(imp, keep, pool_k, chunk, pos0, stream=stream)
    out = gather(tokens, ids, n_kept, stream=stream)
    return dict(importance=imp, ids=ids, pos=pos, n_kept=n_kept, out_tokens=out, first_decode=K.shape[3] + pos0)


def run_host(Qh, Kh, tokens_h, dev: dict, keep, pool_k, chunk, R_valid=None, scale=None, pos0=0, host_out=None,
             stream=None):
    """End to end from host (pinned) buffers through sp_run_host: H2D copies,
    score, select, gather and D2H copies, all enqueued on one stream.
    ``dev`` holds preallocated device tensors Q, K, tokens, importance, ids,
    pos, n_kept, out_tokens, ws (see bench.py)."""
    g, lay = make_geom(dev["Q"], dev["K"], R_valid, scale)
    p = _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))
    ho = host_out
    io = _lib.sp_host_io(Q=Qh.data_ptr(), K=Kh.data_ptr(), tokens=tokens_h.data_ptr(), ids=ho["ids"].data_ptr(),
                         pos=ho["pos"].data_ptr(), n_kept=ho["n_kept"].data_ptr(),
                         out_tokens=ho["out_tokens"].data_ptr(),
                         q_bytes=Qh.numel() * 2, k_bytes=Kh.numel() * 2)
    db = _lib.sp_device_bufs(Q=dev["Q"].data_ptr(), K=dev["K"].data_ptr(), tokens=dev["tokens"].data_ptr(),
                             importance=dev["importance"].data_ptr(), ids=dev["ids"].data_ptr(),
                             pos=dev["pos"].data_ptr(), n_kept=dev["n_kept"].data_ptr(),
                             out_tokens=dev["out_tokens"].data_ptr(), ws=dev["ws"].data_ptr(),
                             ws_bytes=dev["ws"].numel())
    check(lib().sp_run_host(C.byref(io), C.byref(db), C.byref(g), C.byref(lay), C.byref(p), _stream_ptr(stream)),
          "sp_run_host")


def run_workspace_bytes(Q, K, keep, pool_k, chunk, R_valid=None, scale=None, pos0=0) -> int:
    g, _ = make_geom(Q, K, R_valid, scale)
    p = _lib.sp_select_params(keep_rate=float(keep), pool_k=int(pool_k), chunk=int(chunk), pos0=int(pos0))
    return lib().sp_run_workspace_bytes(C.byref(g), C.byref(p))
