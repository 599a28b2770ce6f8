"""Pins for the float64 oracle (CPU only).

Each oracle step is checked against something other than itself: the paper's
worked example, SPEC.md's hand-checked examples, closed forms, library routines
in the special cases that reduce to them, invariants and brute force.  See
DESIGN.md "Oracle pins" for the table.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.special
import torch

from oracle import ref, tiny
from spgen import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rand_qk(rng, L, H, Hkv, N, d, R, dyadic=True):
    """Random f64 inputs on a dyadic grid (exact in bf16 and in f64 sums)."""
    if dyadic:
        Q = rng.integers(-64, 65, size=(L, R, H, d)) / 32.0
        K = rng.integers(-64, 65, size=(L, Hkv, N, d)) / 32.0
    else:
        Q = rng.standard_normal((L, R, H, d))
        K = rng.standard_normal((L, Hkv, N, d))
    return Q, K


# ---------------------------------------------------------------- O9 (paper example)
def test_paper_position_example():
    g = _golden("paper_position_ids.json")
    N, kept = g["N"], np.array(g["kept"])
    ids, pos, first = ref.restore_position_ids(kept, chunk=1, N=N, pos0=0)
    assert list(pos) == g["speculated_pos_ids"]
    decoding = list(pos) + [first + j for j in range(3)]
    assert decoding == g["decoding_pos_ids_prefix"]


def test_gather_paper_example():
    """O10 pinned by the paper's worked example: with the prompt's
    tokens standing for their original positions [0..9], gathering the kept
    tokens [0, 1, 3, 6, 7] must give the "Speculated Pos Ids" row."""
    g = _golden("paper_position_ids.json")
    tokens = np.array(g["original_pos_ids"], dtype=np.int32)
    assert list(ref.gather(tokens, np.array(g["kept"]))) == g["speculated_pos_ids"]


def test_gather_closed_forms():
    """O10 closed forms: tokens[i] = a + b*i gathers to a + b*ids; gathering a
    gather composes the index maps; on the whole path, tokens = arange(N)
    returns the kept ids themselves."""
    rng = np.random.default_rng(7)
    ids = np.sort(rng.choice(1000, size=137, replace=False))
    assert (ref.gather(5 + 3 * np.arange(1000), ids) == 5 + 3 * ids).all()
    tok = rng.integers(0, 128256, size=1000)
    sub = np.sort(rng.choice(137, size=40, replace=False))
    assert (ref.gather(ref.gather(tok, ids), sub) == tok[ids[sub]]).all()
    w = gen.CONFIGS["C0"]
    Qb, Kb, _ = gen.gen_request(w, 0)
    r = ref.specprefill(Qb, Kb, np.arange(w.N, dtype=np.int32), w.scale, w.keep, w.pool_k, w.chunk)
    assert (r["out_tokens"] == r["ids"]).all() and len(r["ids"]) == r["n_kept"]


def test_position_offset_and_partial_chunk():
    ids, pos, first = ref.restore_position_ids(np.array([0, 2]), chunk=4, N=10, pos0=100)
    assert list(ids) == [0, 1, 2, 3, 8, 9]          # chunk 2 is the partial tail [8, 10)
    assert list(pos) == [100, 101, 102, 103, 108, 109]
    assert first == 110


# ---------------------------------------------------------------- O1-O4 closed forms
def test_single_head_equals_library_softmax():
    """L=H=Hkv=R=1: importance is exactly softmax(scale * K q)."""
    rng = np.random.default_rng(0)
    Q, K = _rand_qk(rng, 1, 1, 1, 37, 16, 1, dyadic=False)
    scale = 0.37
    imp = ref.token_importance(Q, K, scale)
    expect = scipy.special.softmax(scale * (K[0, 0] @ Q[0, 0, 0]))
    np.testing.assert_allclose(imp, expect, rtol=1e-13, atol=0)


@pytest.mark.parametrize("scale", [1.0, 1.0 / math.sqrt(16)])
def test_one_needle_closed_form(scale):
    """q = e0, k_3 = 2 e0, other keys 0, N = 10: imp[3] = e^{2s}/(e^{2s}+9)."""
    N, d = 10, 16
    Q = np.zeros((1, 1, 1, d)); Q[0, 0, 0, 0] = 1.0
    K = np.zeros((1, 1, N, d)); K[0, 0, 3, 0] = 2.0
    imp = ref.token_importance(Q, K, scale)
    e = math.exp(2 * scale)
    assert imp[3] == pytest.approx(e / (e + 9), rel=1e-14)
    for i in range(N):
        if i != 3:
            assert imp[i] == pytest.approx(1 / (e + 9), rel=1e-14)


def test_gqa_mapping_closed_form():
    """H=4, Hkv=2: q heads {0,1} read kv head 0, heads {2,3} read kv head 1 (Z4).
    Heads 0 and 1 are aligned with a needle at token 3 of kv head 0; kv head 1
    has a needle at token 7 that no aligned head sees.  Closed form:
    imp[3] = e^2/(e^2+N-1), every other token 1/N (the q=0 heads)."""
    N, d = 12, 16
    Q = np.zeros((1, 1, 4, d)); Q[0, 0, 0, 0] = 1.0; Q[0, 0, 1, 0] = 1.0
    K = np.zeros((1, 2, N, d)); K[0, 0, 3, 0] = 2.0; K[0, 1, 7, 0] = 2.0
    imp = ref.token_importance(Q, K, 1.0)
    e2 = math.exp(2.0)
    assert imp[3] == pytest.approx(e2 / (e2 + N - 1), rel=1e-14)
    assert imp[7] == pytest.approx(1.0 / N, rel=1e-14)
    for i in set(range(N)) - {3, 7}:
        assert imp[i] == pytest.approx(1.0 / N, rel=1e-14)


def test_uniform_closed_forms():
    rng = np.random.default_rng(1)
    Q, K = _rand_qk(rng, 2, 4, 2, 9, 8, 3)
    K_eq = np.repeat(K[:, :, :1, :], 9, axis=2)              # all keys equal
    np.testing.assert_allclose(ref.token_importance(Q, K_eq, 0.5), np.full(9, 1 / 9), rtol=1e-14)
    np.testing.assert_allclose(ref.token_importance(np.zeros_like(Q), K, 0.5), np.full(9, 1 / 9), rtol=1e-14)


def test_spec_aggregation_example():
    g = _golden("spec_examples.json")["aggregation"]
    # SPEC's tensor is [rows][L][S][H], the paper's [N, L, S, H] layout
    A = np.array(g["attn"], dtype=np.float64)
    assert list(A.shape) == g["shape"]
    np.testing.assert_allclose(ref.aggregate_attention(A), g["expected"], rtol=1e-15)


def test_masked_row_equals_valid_row_alone():
    """one of two rows invalid -> the valid row's max-reduction alone."""
    rng = np.random.default_rng(2)
    A = rng.random((2, 3, 5, 4))
    np.testing.assert_array_equal(ref.aggregate_attention(A, R_valid=1), A[0].max(axis=2).max(axis=0))
    with pytest.raises(ValueError):
        ref.aggregate_attention(A, R_valid=0)


def test_rows_sum_to_one():
    """Every (layer, head, row) softmax sums to 1 over the prompt (BJ invariant)."""
    rng = np.random.default_rng(3)
    Q, K = _rand_qk(rng, 2, 4, 2, 33, 16, 3, dyadic=False)
    A = ref.attention_scores(Q, K, 0.25)
    np.testing.assert_allclose(A.sum(axis=2), 1.0, rtol=1e-13)
    assert (A >= 0).all()


def test_importance_sum_bounds():
    """1 <= sum_i imp <= L*H (sum of maxima >= max of sums = 1; <= sum of all
    L*H rows); equality at 1 when all (l, h) rows are identical."""
    rng = np.random.default_rng(4)
    Q, K = _rand_qk(rng, 3, 4, 2, 50, 16, 2, dyadic=False)
    s = ref.token_importance(Q, K, 0.3).sum()
    assert 1.0 - 1e-12 <= s <= 3 * 4 + 1e-12
    Qs = np.repeat(Q[:1, :, :1], 3, axis=0).repeat(4, axis=2)
    Ks = np.repeat(K[:1, :1], 3, axis=0).repeat(2, axis=1)
    assert ref.token_importance(Qs, Ks, 0.3).sum() == pytest.approx(1.0, rel=1e-13)


def test_shift_invariance():
    """K[l, g, :, :] += v (same v for every token) leaves imp unchanged."""
    rng = np.random.default_rng(5)
    Q, K = _rand_qk(rng, 2, 4, 2, 40, 16, 2)
    v = rng.integers(-8, 9, size=(2, 2, 1, 16)) / 8.0
    np.testing.assert_allclose(ref.token_importance(Q, K + v, 0.25), ref.token_importance(Q, K, 0.25), rtol=1e-11)


def test_permutation_symmetries():
    rng = np.random.default_rng(6)
    L, H, Hkv, N, d, R = 3, 6, 3, 25, 8, 2
    Q, K = _rand_qk(rng, L, H, Hkv, N, d, R, dyadic=False)
    base = ref.token_importance(Q, K, 0.5)
    p = rng.permutation(N)                                   # token permutation: equivariant
    np.testing.assert_allclose(ref.token_importance(Q, K[:, :, p], 0.5), base[p], rtol=1e-13)
    pl = rng.permutation(L)                                  # layer permutation: invariant
    np.testing.assert_allclose(ref.token_importance(Q[pl], K[pl], 0.5), base, rtol=1e-13)
    G = H // Hkv                                             # kv head together with its q group
    pg = rng.permutation(Hkv)
    ph = np.concatenate([np.arange(g * G, (g + 1) * G) for g in pg])
    np.testing.assert_allclose(ref.token_importance(Q[:, :, ph], K[:, pg], 0.5), base, rtol=1e-13)


def test_r_valid_prefix():
    rng = np.random.default_rng(7)
    Q, K = _rand_qk(rng, 2, 4, 2, 30, 16, 4)
    np.testing.assert_array_equal(ref.token_importance(Q, K, 0.25, R_valid=2),
                                  ref.token_importance(Q[:, :2], K, 0.25))


def test_streamed_equals_materialised():
    rng = np.random.default_rng(8)
    Q, K = _rand_qk(rng, 3, 4, 2, 21, 16, 3, dyadic=False)
    A = ref.attention_scores(Q, K, 0.25)
    np.testing.assert_allclose(ref.token_importance(Q, K, 0.25), ref.aggregate_attention(A), rtol=1e-15)
    np.testing.assert_allclose(ref.token_importance(Q, lambda l: K[l], 0.25), ref.aggregate_attention(A), rtol=1e-15)


# ---------------------------------------------------------------- O5 pooling
def test_pooling_examples():
    for ex in _golden("spec_examples.json")["pooling"]:
        np.testing.assert_allclose(ref.smooth_scores(np.array(ex["x"], float), ex["pool_k"]), ex["expected"], rtol=1e-15)


def test_pooling_identity_constant_and_errors():
    rng = np.random.default_rng(9)
    x = rng.random(17)
    np.testing.assert_array_equal(ref.smooth_scores(x, 1), x)
    np.testing.assert_allclose(ref.smooth_scores(np.full(11, 0.3), 5), 0.3, rtol=1e-15)
    for bad in (0, 2, 4, -1):
        with pytest.raises(ValueError):
            ref.smooth_scores(x, bad)


@pytest.mark.parametrize("pool_k", [3, 5, 7, 9])
def test_pooling_vs_torch_and_fractions(pool_k):
    """Shrinking-window mean == torch avg_pool1d(count_include_pad=False) in f64,
    and == the exact Fraction mean."""
    rng = np.random.default_rng(pool_k)
    x = rng.random(23)
    w = (pool_k - 1) // 2
    t = torch.nn.functional.avg_pool1d(torch.tensor(x)[None, None], pool_k, stride=1, padding=w,
                                       count_include_pad=False)[0, 0].numpy()
    got = ref.smooth_scores(x, pool_k)
    np.testing.assert_allclose(got, t, rtol=1e-14)
    np.testing.assert_allclose(got, [float(f) for f in tiny.pooled_exact(x, pool_k)], rtol=1e-15)


# ---------------------------------------------------------------- O6 chunk means
@pytest.mark.parametrize("N,chunk", [(10, 2), (11, 4), (64, 4), (5, 32), (100, 7), (33, 1)])
def test_chunk_scores_vs_torch(N, chunk):
    rng = np.random.default_rng(N * 100 + chunk)
    x = rng.random(N)
    t = torch.nn.functional.avg_pool1d(torch.tensor(x)[None, None], chunk, stride=chunk, ceil_mode=True,
                                       count_include_pad=False)[0, 0].numpy()
    np.testing.assert_allclose(ref.chunk_scores(x, chunk), t, rtol=1e-14)


def test_partial_chunk_example():
    np.testing.assert_array_equal(ref.chunk_scores(np.array([1, 1, 1, 1, 8.0]), 2), [1, 1, 8])


# ---------------------------------------------------------------- O7 budget
def test_count_example():
    g = _golden("spec_examples.json")["count"]
    n_c = -(-g["N"] // g["chunk"])
    assert ref.kept_chunk_count(n_c, g["keep"]) * g["chunk"] == g["expected_tokens"]


def test_count_matches_exact_rational_ceil():
    """K_c = max(1, ceil(keep * n_c)) with keep read as the decimal it is written as."""
    for keep_s in ["0.1", "0.2", "0.3", "0.25", "0.5", "0.6", "0.7", "0.9", "1", "0.001", "0.999999", "0.123456"]:
        keep = float(keep_s)
        for n_c in [1, 2, 3, 7, 10, 16, 25, 50, 128, 1000, 1024, 4096, 131072]:
            exact = max(1, math.ceil(Fraction(keep_s) * n_c))
            assert ref.kept_chunk_count(n_c, keep) == min(n_c, exact), (keep_s, n_c)
    # computed keep values (i/10.0) used by the C4 sweep
    table = [410, 820, 1229, 1639, 2048, 2458, 2868, 3277, 3687]
    assert [ref.kept_chunk_count(4096, i / 10.0) for i in range(1, 10)] == table
    assert ref.kept_chunk_count(16, 0.5) == 8                 # C0: 8 chunks of 4 = 32 tokens = ceil(0.5*64)
    for bad in (0.0, -0.1, 1.0000001, 2.0):
        with pytest.raises(ValueError):
            ref.kept_chunk_count(10, bad)


# ---------------------------------------------------------------- O8 top-K
def test_chunk_select_example():
    g = _golden("spec_examples.json")["chunk_select"]
    r = ref.select(np.array(g["scores"], float), g["keep"], pool_k=1, chunk=g["chunk"])
    np.testing.assert_array_equal(r["cs"], g["chunk_means"])
    assert list(r["ids"]) == g["expected_ids"]


@pytest.mark.parametrize("seed", range(12))
def test_topk_bruteforce(seed):
    """Kept set == lexicographically smallest max-sum K-subset (exact sums),
    on dyadic scores with many exact ties."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 13))
    cs = rng.integers(0, 5, size=n) / 4.0
    for K in range(1, n + 1):
        assert list(ref.select_chunks(cs, K)) == tiny.topk_bruteforce(cs, K)


def test_c0_sized_bruteforce():
    """C0 has 16 chunks and keeps 8: C(16, 8) = 12,870 subsets."""
    rng = np.random.default_rng(123)
    cs = rng.integers(0, 6, size=16) / 8.0
    assert list(ref.select_chunks(cs, 8)) == tiny.topk_bruteforce(cs, 8)


def test_topk_nesting_and_scale_invariance():
    rng = np.random.default_rng(10)
    cs = rng.integers(0, 20, size=200) / 16.0
    prev = set()
    for i in range(1, 11):
        kept = set(ref.select_chunks(cs, ref.kept_chunk_count(200, i / 10.0)))
        assert prev <= kept
        prev = kept
    for p2 in (0.25, 2.0, 1024.0):
        np.testing.assert_array_equal(ref.select_chunks(cs * p2, 37), ref.select_chunks(cs, 37))


def test_keep_one_keeps_everything_and_short_prompt():
    rng = np.random.default_rng(11)
    imp = rng.random(50)
    assert list(ref.select(imp, 1.0, 3, 8)["ids"]) == list(range(50))
    r = ref.select(rng.random(3), 0.1, 5, 32)                 # M < chunk: a single chunk, kept
    assert list(r["ids"]) == [0, 1, 2]


# ---------------------------------------------------------------- whole path
def test_planted_needle_kept():
    """A chunk whose keys align with the look-ahead queries is kept at keep 0.1
    for every seed."""
    L, H, Hkv, N, d, R, chunk = 2, 4, 2, 640, 32, 2, 32
    for seed in range(5):
        rng = np.random.default_rng(seed)
        Q = rng.integers(-16, 17, size=(L, R, H, d)) / 16.0
        K = rng.integers(-16, 17, size=(L, Hkv, N, d)) / 16.0
        c = int(rng.integers(1, N // chunk))
        G = H // Hkv
        for l in range(L):
            for g in range(Hkv):
                K[l, g, c * chunk:(c + 1) * chunk] += 0.5 * Q[l, 0, g * G][None, :]
        r = ref.select(ref.token_importance(Q, K, 1 / math.sqrt(d)), 0.1, 5, chunk)
        assert c in set(r["kept_chunks"]), (seed, c)


def test_gather_and_invariants_on_c0():
    w = gen.CONFIGS["C0"]
    Qb, Kb, tok = gen.gen_request(w, 0)
    r = ref.specprefill(Qb, Kb, tok, w.scale, w.keep, w.pool_k, w.chunk)
    ids = r["ids"]
    assert (np.diff(ids) > 0).all()                          # strictly ascending
    assert r["n_kept"] == 32 == math.ceil(w.keep * w.N)       # BJ token law (holds for C0)
    for j, i in enumerate(ids):
        assert r["out_tokens"][j] == tok[i]
    assert r["first_decode"] == w.N
    assert 1.0 - 1e-12 <= r["imp"].sum() <= w.L * w.H


def test_margin():
    assert ref.margin(np.array([3.0, 2.0, 1.0]), 3) == math.inf
    assert ref.margin(np.array([3.0, 2.0, 1.0]), 1) == pytest.approx(1 / 3)
    assert ref.margin(np.array([2.0, 2.0, 1.0]), 1) == 0.0


# ---------------------------------------------------------------- O2 normaliser (row f2 hand-over)
def test_softmax_lse_closed_forms_and_library():
    """lse pins: uniform keys (all logits equal c) give c + ln N; the needle case
    gives ln(e^{2s} + N - 1); in general it equals scipy's logsumexp of the
    logits, and exp(s - lse) rows sum to one."""
    N, d = 10, 16
    Q = np.zeros((1, 1, 1, d)); Q[0, 0, 0, 0] = 1.0
    K = np.zeros((1, 1, N, d)); K[0, 0, 3, 0] = 2.0
    lse = ref.softmax_lse(Q, K, 0.5)
    assert lse[0, 0, 0] == pytest.approx(math.log(math.exp(1.0) + N - 1), rel=1e-15)
    K1 = np.zeros((1, 1, N, d)); K1[0, 0, :, 0] = 3.0            # every logit = 0.5 * 3
    assert ref.softmax_lse(Q, K1, 0.5)[0, 0, 0] == pytest.approx(1.5 + math.log(N), rel=1e-15)
    rng = np.random.default_rng(11)
    Q, K = _rand_qk(rng, 2, 4, 2, 33, 8, 3, dyadic=False)
    lse = ref.softmax_lse(Q, K, 0.3)
    for l in range(2):
        for h in range(4):
            s = 0.3 * (Q[l, :, h, :] @ K[l, h // 2].T)
            np.testing.assert_allclose(lse[l, h], scipy.special.logsumexp(s, axis=1), rtol=1e-14)
            np.testing.assert_allclose(np.exp(s - lse[l, h][:, None]).sum(axis=1), 1.0, rtol=1e-13)


# ------------------------------------------------------------------ row f4: e4m3 decoder
def test_e4m3_decoder_format_values():
    """Values the OCP E4M3 definition fixes: 1.0 = 0x38, max normal 448 = 0x7E,
    min normal 2^-6 = 0x08, min subnormal 2^-9 = 0x01, -2 = 0xC0, NaN = 0x7F/0xFF."""
    c = np.array([0x00, 0x80, 0x38, 0x7E, 0x08, 0x01, 0x07, 0xC0, 0x3C, 0x77], dtype=np.uint8)
    want = [0.0, -0.0, 1.0, 448.0, 2.0 ** -6, 2.0 ** -9, 7 * 2.0 ** -9, -2.0, 1.5, 240.0]
    np.testing.assert_array_equal(ref.e4m3_to_f64(c), want)
    assert np.isnan(ref.e4m3_to_f64(np.array([0x7F, 0xFF], dtype=np.uint8))).all()


def test_e4m3_decoder_vs_torch_all_codes():
    """All 256 codes against torch's float8_e4m3fn (a library decoder)."""
    codes = np.arange(256, dtype=np.uint8)
    lib = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    mine = ref.e4m3_to_f64(codes)
    nan = np.isnan(lib)
    np.testing.assert_array_equal(np.isnan(mine), nan)
    np.testing.assert_array_equal(mine[~nan], lib[~nan])


def test_e4m3_path_equals_bf16_path_on_common_values():
    """Values exactly representable in both formats give the same importance
    through specprefill_e4m3 (with scales) and specprefill (bf16)."""
    rng = np.random.default_rng(5)
    L, R, H, Hkv, N, d = 2, 2, 4, 2, 24, 16
    codes_q = rng.integers(0x30, 0x48, size=(L, R, H, d)).astype(np.uint8) | (rng.integers(0, 2, (L, R, H, d)) << 7).astype(np.uint8)
    codes_k = rng.integers(0x28, 0x48, size=(L, Hkv, N, d)).astype(np.uint8)
    Qv = 0.5 * ref.e4m3_to_f64(codes_q)
    Kv = 0.25 * ref.e4m3_to_f64(codes_k)
    to_bits = lambda x: (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)   # exact: <= 4 significant bits
    tokens = np.arange(N)
    a = ref.specprefill_e4m3(codes_q, codes_k, 0.5, 0.25, tokens, 0.25, 0.5, 3, 4)
    b = ref.specprefill(to_bits(Qv), to_bits(Kv), tokens, 0.25, 0.5, 3, 4)
    np.testing.assert_array_equal(a["imp"], b["imp"])
    np.testing.assert_array_equal(a["ids"], b["ids"])


# ------------------------------------------------------------------ row f4: look-ahead-key denominator (Z2')
def test_lookahead_denominator_closed_form():
    """All logits equal (Q = 0): every visible key has probability 1/(N + n_la(r)),
    so the importance of each prompt token is mean_r 1/(N + r + 1 - shift)."""
    L, R, H, Hkv, N, d = 2, 3, 4, 2, 10, 8
    Q = np.zeros((L, R, H, d))
    rng = np.random.default_rng(0)
    K = rng.normal(size=(L, Hkv, N, d))
    K_la = rng.normal(size=(L, Hkv, R, d))
    for shift in (0, 1):
        A = ref.attention_scores_lookahead(Q, K, K_la, 0.5, shift)
        imp = ref.aggregate_attention(A)
        want = np.mean([1.0 / (N + max(0, r + 1 - shift)) for r in range(R)])
        np.testing.assert_allclose(imp, want, rtol=1e-14)


def test_lookahead_denominator_vs_library_softmax():
    """One (l, h, r) slice equals scipy's softmax over the concatenated key set,
    sliced to the prompt entries; prompt + look-ahead probabilities sum to 1."""
    rng = np.random.default_rng(1)
    L, R, H, Hkv, N, d = 1, 4, 2, 1, 7, 5
    Q, K, K_la = rng.normal(size=(L, R, H, d)), rng.normal(size=(L, Hkv, N, d)), rng.normal(size=(L, Hkv, R, d))
    A = ref.attention_scores_lookahead(Q, K, K_la, 0.7, 0)
    for r in range(R):
        for h in range(H):
            keys = np.concatenate([K[0, 0], K_la[0, 0, :r + 1]])
            p = scipy.special.softmax(0.7 * keys @ Q[0, r, h])
            np.testing.assert_allclose(A[r, 0, :, h], p[:N], rtol=1e-13)
            assert A[r, 0, :, h].sum() < 1.0


def test_lookahead_denominator_shift_one_row0_is_plain():
    """la_shift = 1: row 0 sees no look-ahead key, so it equals the plain (Z2) row."""
    rng = np.random.default_rng(2)
    L, R, H, Hkv, N, d = 2, 3, 4, 2, 9, 6
    Q, K, K_la = rng.normal(size=(L, R, H, d)), rng.normal(size=(L, Hkv, N, d)), rng.normal(size=(L, Hkv, R, d))
    A1 = ref.attention_scores_lookahead(Q, K, K_la, 0.3, 1)
    A0 = ref.attention_scores(Q, K, 0.3)
    np.testing.assert_allclose(A1[0], A0[0], rtol=1e-13)
    assert (A1[1:] < A0[1:]).all()
