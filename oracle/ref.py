"""SpecPrefill float64 CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The CUDA path never imports,
links or calls it, and it shares no code with ``paper_2502_02789_b200/``.

It is a plain, slow, step-by-step transcription of the method of
arXiv 2502.02789 ("SpecPrefill"), in float64, following the paper's order and
notation.  Citations: ``P:n`` = line n of the paper's LaTeX, with
the section label; ``S:n`` = line n of SPEC.md (interface/test ideas only);
``Zk`` = reading k in DESIGN.md's ambiguity register.

Pins (tests/test_oracle.py): every function below is checked against something
other than itself -- the paper's worked example, SPEC's hand-checked examples,
closed forms, library routines in special cases, invariants and brute force.
No function here is "parity unpinned".

Conventions
-----------
* Inputs arrive as bf16 bit patterns (uint16) and are widened exactly to f64.
* Shapes (one request): Q [L][R][H][d], K [L][Hkv][N][d].  GQA: query head h
  reads kv head h // G with G = H / Hkv (Z4).
"""
from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------------ inputs
def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact bf16 -> float64 (bf16 is the top half of an IEEE float32)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def e4m3_to_f64(codes: np.ndarray) -> np.ndarray:
    """Exact OCP FP8 E4M3 ("e4m3fn") -> float64, from the format's definition
    (an FP8 KV cache): bit 7 sign, bits 6..3 exponent E with
    bias 7, bits 2..0 mantissa M.  E > 0: (-1)^s * 2^(E-7) * (1 + M/8);
    E = 0: (-1)^s * 2^-6 * (M/8) (subnormal); S.1111.111 is NaN; no infinities
    (so E = 15 with M < 7 is a normal number, max 448)."""
    c = np.asarray(codes, dtype=np.uint8).astype(np.int64)
    sign = np.where(c >> 7, -1.0, 1.0)
    E = (c >> 3) & 15
    M = (c & 7).astype(np.float64)
    mag = np.where(E > 0, np.ldexp(1.0 + M / 8.0, (E - 7).astype(np.int32)), np.ldexp(M / 8.0, -6))
    out = sign * mag
    return np.where((c & 0x7F) == 0x7F, np.nan, out)


# ------------------------------------------------------------------ O1-O2
def attention_scores(Q: np.ndarray, K: np.ndarray, scale: float) -> np.ndarray:
    """Speculator attention of the look-ahead rows over the prompt, one request.

    P:103-107 (sec:token_importance, eq.):  a_ij := Softmax(Q_{M+j} K^T)_i,
    0 <= i < M (prompt tokens), 0 <= j < N (look-ahead rows), per layer (and,
    as in any multi-head attention, per head).  Here rows j are ``r`` (Z1),
    the softmax runs over the prompt keys only (Z2) and the logits carry the
    attention scale (Z3).

    Q [L][R][H][d] f64, K [L][Hkv][N][d] f64  ->  A [R][L][N][H] f64
    (the paper's [N, L, S, H] attention tensor of sec:attn_agg).
    """
    L, R, H, d = Q.shape
    Lk, Hkv, N, dk = K.shape
    assert L == Lk and d == dk and H % Hkv == 0
    G = H // Hkv
    A = np.empty((R, L, N, H), dtype=np.float64)
    for l in range(L):
        for h in range(H):
            k = K[l, h // G]                       # [N][d]   GQA: kv head h // G (Z4)
            s = scale * (Q[l, :, h, :] @ k.T)      # [R][N]   O1 logits
            m = s.max(axis=1, keepdims=True)       # O2 softmax over the prompt keys
            e = np.exp(s - m)
            A[:, l, :, h] = e / e.sum(axis=1, keepdims=True)
    return A


def softmax_lse(Q: np.ndarray, K: np.ndarray, scale: float) -> np.ndarray:
    """O2's normaliser on its own: lse[l][h][r] = ln sum_i exp(s[l,h,r,i]) over
    the prompt keys (Z2), s as in O1.  This is the per-row log-sum-exp
    an attention kernel of the speculator returns: given it,
    the softmax of O2 is exp(s - lse).

    Q [L][R][H][d] f64, K [L][Hkv][N][d] f64 -> lse [L][H][R] f64.
    """
    L, R, H, d = Q.shape
    G = H // K.shape[1]
    out = np.empty((L, H, R), dtype=np.float64)
    for l in range(L):
        for h in range(H):
            s = scale * (Q[l, :, h, :] @ K[l, h // G].T)      # [R][N]
            m = s.max(axis=1)
            out[l, h] = m + np.log(np.exp(s - m[:, None]).sum(axis=1))
    return out


def attention_scores_lookahead(Q: np.ndarray, K: np.ndarray, K_la: np.ndarray, scale: float,
                               la_shift: int = 0) -> np.ndarray:
    """Reading Z2' ("softmax over ALL keys visible
    to that row (context plus any earlier decoded tokens) ... sliced to the first
    M context entries WITHOUT renormalization"): look-ahead row r attends to the
    N prompt keys and to the look-ahead tokens' keys K_la[j], j <= r - la_shift
    (causal; la_shift = 0: row r's own key is K_la[r]; 1: row 0 is the last
    prompt token and sees none).  The softmax runs over that whole key set and
    is then sliced to the prompt entries (P:105-107's a_ij, i < M).

    Q [L][R][H][d], K [L][Hkv][N][d], K_la [L][Hkv][R][d]  ->  A [R][L][N][H].
    """
    L, R, H, d = Q.shape
    Hkv, N = K.shape[1], K.shape[2]
    G = H // Hkv
    A = np.empty((R, L, N, H), dtype=np.float64)
    for l in range(L):
        for h in range(H):
            for r in range(R):
                n_la = max(0, r + 1 - la_shift)
                keys = np.concatenate([K[l, h // G], K_la[l, h // G, :n_la]], axis=0)   # prompt, then look-ahead
                s = scale * (keys @ Q[l, r, h])
                e = np.exp(s - s.max())
                A[r, l, :, h] = e[:N] / e.sum()                    # slice, no renormalisation
    return A


# ------------------------------------------------------------------ O3-O4
def aggregate_attention(A: np.ndarray, R_valid: int | None = None) -> np.ndarray:
    """Max-mean aggregation, P:117-119 (sec:attn_agg): "take the maximum over H
    and L dimension ... and average over N" (N = look-ahead rows).  Only the
    first ``R_valid`` rows are valid (EOS check, Alg.1; Z13).

    A [R][L][N][H] -> importance [N] (token importance vector, length S).
    """
    R = A.shape[0]
    Rv = R if R_valid is None else R_valid
    if Rv < 1:
        raise ValueError("zero valid look-ahead rows (S:182)")
    mx = A[:Rv].max(axis=3).max(axis=1)           # max over H, then over L -> [Rv][N]
    return mx.mean(axis=0)                         # mean over valid rows -> [N]


def token_importance(Q: np.ndarray, K: np.ndarray, scale: float, R_valid: int | None = None) -> np.ndarray:
    """O1-O4 for one request.  Materialises the attention tensor one layer at a
    time (max over L taken across layers, which is exact in any order) so the
    8B-shaped configs fit in host memory.  ``K`` is [L][Hkv][N][d] f64 or a
    callable ``l -> [Hkv][N][d]`` f64."""
    L = Q.shape[0]
    R = Q.shape[1]
    Rv = R if R_valid is None else R_valid
    K_layer = K if callable(K) else (lambda l: K[l])                  # K may be generated per layer
    best = None
    for l in range(L):
        A_l = attention_scores(Q[l:l + 1, :Rv], K_layer(l)[None], scale)   # [Rv][1][N][H]
        m_l = A_l.max(axis=3)[:, 0, :]                               # max over H -> [Rv][N]
        best = m_l if best is None else np.maximum(best, m_l)        # max over L
    return best.mean(axis=0)


# ------------------------------------------------------------------ O5
def smooth_scores(imp: np.ndarray, pool_k: int) -> np.ndarray:
    """1-D average pooling before chunking, P:123 (sec:chunk_select): "we apply a
    1D average pooling before this to smooth the cross block scores".
    Odd window, stride 1, centred, shrinking window at the edges (Z6).
    """
    if pool_k < 1 or pool_k % 2 == 0:
        raise ValueError("pool_k must be odd and >= 1 (S:190)")
    N = len(imp)
    w = (pool_k - 1) // 2
    out = np.empty(N, dtype=np.float64)
    for i in range(N):
        lo, hi = max(0, i - w), min(N - 1, i + w)
        out[i] = imp[lo:hi + 1].sum() / (hi - lo + 1)
    return out


# ------------------------------------------------------------------ O6
def chunk_scores(pooled: np.ndarray, chunk: int) -> np.ndarray:
    """P:121-123 (sec:chunk_select): "we chunk the context contiguously and
    average the token score within each block".  The partial last chunk is
    averaged over its true size (Z8)."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    N = len(pooled)
    n_c = -(-N // chunk)
    return np.array([pooled[c * chunk:min(N, (c + 1) * chunk)].mean() for c in range(n_c)], dtype=np.float64)


# ------------------------------------------------------------------ O7
def kept_chunk_count(n_chunks: int, keep: float) -> int:
    """Budget: the keep rate is "the ratio of chunks", K = max(1,
    ceil(keep * n_chunks)).  Evaluated exactly on keep snapped to
    parts per million (Z9): ppm = floor(keep*1e6 + 0.5); K = ceil(ppm*n/1e6)."""
    if not (0.0 < keep <= 1.0):
        raise ValueError("keep_rate must be in (0, 1] (S:145)")
    ppm = int(math.floor(keep * 1_000_000 + 0.5))
    k = (ppm * n_chunks + 999_999) // 1_000_000
    return max(1, min(n_chunks, k))


# ------------------------------------------------------------------ O8
def select_chunks(cs: np.ndarray, K_c: int) -> np.ndarray:
    """"then we select the Top-K blocks".  Order by (score desc, index
    asc) -- lowest index wins ties (Z10) -- keep the first K_c, return the
    kept chunk indices ascending (Z11)."""
    n_c = len(cs)
    order = np.lexsort((np.arange(n_c), -cs))      # primary key -cs, secondary index
    return np.sort(order[:K_c])


# ------------------------------------------------------------------ O9
def restore_position_ids(kept_chunks: np.ndarray, chunk: int, N: int, pos0: int = 0):
    """sec:position_ids: kept tokens keep their original position ids
    (non-contiguous), and the first decoding position is the context length
    ("explicitly set the decoding token position to the context length").
    Worked example P:129-131.  Returns (ids, pos, first_decode)."""
    ids = [t for c in kept_chunks for t in range(c * chunk, min(N, (c + 1) * chunk))]
    ids = np.array(ids, dtype=np.int64)
    return ids, ids + pos0, N + pos0


# ------------------------------------------------------------------ O10
def gather(tokens: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """merge_requests input (Alg.1): the selected tokens, in order."""
    return np.asarray(tokens)[np.asarray(ids, dtype=np.int64)]


# ------------------------------------------------------------------ whole path
def select(imp: np.ndarray, keep: float, pool_k: int, chunk: int, pos0: int = 0) -> dict:
    """O5-O9 for one request (Alg.1)."""
    pooled = smooth_scores(imp, pool_k)
    cs = chunk_scores(pooled, chunk)
    K_c = kept_chunk_count(len(cs), keep)
    kept = select_chunks(cs, K_c)
    ids, pos, first = restore_position_ids(kept, chunk, len(imp), pos0)
    return dict(pooled=pooled, cs=cs, K_c=K_c, kept_chunks=kept, ids=ids, pos=pos,
                first_decode=first, n_kept=len(ids))


def specprefill(Q_bits, K_bits, tokens, scale, keep, pool_k, chunk, R_valid=None, pos0=0) -> dict:
    """Full hot path for one request: Alg.1 P:158-166 (retrieve_qk ->
    compute_attention_score -> aggregate -> chunk_select -> restore_pos_ids ->
    merge)."""
    Q = bf16_to_f64(Q_bits)
    K = bf16_to_f64(K_bits)
    imp = token_importance(Q, K, scale, R_valid)
    out = select(imp, keep, pool_k, chunk, pos0)
    out["imp"] = imp
    out["out_tokens"] = gather(tokens, out["ids"])
    return out


def specprefill_e4m3(Q_codes, K_codes, q_scale, k_scale, tokens, scale, keep, pool_k, chunk, R_valid=None,
                     pos0=0) -> dict:
    """Row f4: the same path on FP8 inputs.  The dequantised values
    Q = q_scale * e4m3(Q8), K = k_scale * e4m3(K8) are the speculator's query
    rows and keys; everything after is ``specprefill``'s definition."""
    Q = q_scale * e4m3_to_f64(Q_codes)
    K = k_scale * e4m3_to_f64(K_codes)
    imp = token_importance(Q, K, scale, R_valid)
    out = select(imp, keep, pool_k, chunk, pos0)
    out["imp"] = imp
    out["out_tokens"] = gather(tokens, out["ids"])
    return out


def margin(cs: np.ndarray, K_c: int) -> float:
    """Relative gap between the K_c-th and (K_c+1)-th largest chunk score
    (DESIGN.md parity rule); inf when every chunk is kept."""
    if K_c >= len(cs):
        return math.inf
    s = np.sort(cs)[::-1]
    if s[K_c - 1] == 0.0:
        return 0.0
    return float((s[K_c - 1] - s[K_c]) / s[K_c - 1])
