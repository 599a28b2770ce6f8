"""CPU checks of the C ABI boundary: the library loads, exports every symbol
include/specprefill.h declares, and validates arguments on the host (no
compute is launched without a GPU)."""
import ctypes as C
import math
import os
import re

import pytest

import paper_2502_02789_b200 as sp
from paper_2502_02789_b200 import _lib
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "specprefill.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported_and_bound():
    names = _declared()
    assert len(names) >= 15
    h = C.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(h, n), f"{n} declared in specprefill.h but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no Python binding"
    assert set(_lib.SIGNATURES) == set(names)
    assert sp.lib().sp_abi_version() == 1


def test_spgen_library_exports():
    h = C.CDLL(os.path.join(ROOT, "spgen", "libspgen.so"))
    for n in ("spgen_fill_K", "spgen_fill_Q", "spgen_fill_tokens"):
        assert hasattr(h, n)


def test_status_strings():
    for code in (0, 1, 2, 3, 5, 6, 7, 8):
        assert sp.lib().sp_status_string(code).startswith(b"SP_")


def test_kept_chunks_matches_oracle_rule():
    L = sp.lib()
    for keep in [0.001, 0.1, 0.2, 0.25, 0.3, 0.5, 0.6, 0.7, 0.9, 1.0] + [i / 10.0 for i in range(1, 11)]:
        for n in [1, 2, 3, 7, 16, 25, 50, 128, 1024, 4096, 131072]:
            assert L.sp_kept_chunks(n, keep) == ref.kept_chunk_count(n, keep)
    assert L.sp_kept_chunks(10, 0.0) == -1 and L.sp_kept_chunks(10, 1.5) == -1 and L.sp_kept_chunks(0, 0.5) == -1


def _geom(**kw):
    d = dict(B=1, L=2, H=4, Hkv=2, d=16, R=2, R_valid=2, N=64, scale=0.25)
    d.update(kw)
    return _lib.sp_geom(**d)


def _layout(g):
    N, d = g.N, g.d
    return _lib.sp_layout(k_b=g.L * g.Hkv * N * d, k_l=g.Hkv * N * d, k_g=N * d, k_i=d,
                          q_b=g.L * g.R * g.H * d, q_l=g.R * g.H * d, q_r=g.H * d, q_h=d)


FAKE = 1 << 20          # aligned fake device pointers: validation fails before any use


@pytest.mark.parametrize("kw,code", [
    (dict(d=15), _lib.SP_EINVAL), (dict(d=8), _lib.SP_EINVAL), (dict(d=272), _lib.SP_EINVAL),
    (dict(H=5), _lib.SP_EINVAL), (dict(N=0), _lib.SP_EINVAL), (dict(R_valid=3), _lib.SP_EINVAL),
    (dict(R_valid=0), _lib.SP_EEMPTY), (dict(scale=float("nan")), _lib.SP_EINVAL), (dict(scale=0.0), _lib.SP_EINVAL),
    (dict(B=0), _lib.SP_EINVAL),
])
def test_score_validation(kw, code):
    g = _geom(**kw)
    lay = _layout(_geom())
    rc = sp.lib().sp_score(FAKE, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None)
    assert rc == code


def test_score_layout_validation():
    g = _geom()
    lay = _layout(g)
    lay.k_i = 12                                         # 24 B: not a multiple of 16 B
    assert sp.lib().sp_score(FAKE, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    lay = _layout(g)
    assert sp.lib().sp_score(FAKE + 2, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    lay.k_g = -16
    assert sp.lib().sp_score(FAKE, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    assert sp.lib().sp_score(FAKE, FAKE, None, C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL


@pytest.mark.parametrize("field", ["k_b", "k_l", "k_g", "q_b", "q_l", "q_r", "q_h"])
def test_broadcast_strides_rejected(field):
    """A stride-0 (broadcast, e.g. K.expand(B, ...)) dimension of size > 1 is
    rejected on the host for every algorithm (the TMA tensor maps cannot
    express it); stride 0 on a size-1 dimension is irrelevant and accepted."""
    g = _geom(B=2)
    lay = _layout(g)
    setattr(lay, field, 0)
    for algo in (_lib.SP_SCORE_FUSED, _lib.SP_SCORE_SIMT, _lib.SP_SCORE_AUTO):
        assert sp.lib().sp_score_ex(FAKE, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, algo, None) \
            == _lib.SP_EINVAL
    g1 = _geom(B=1)
    lay1 = _layout(g1)
    lay1.k_b = lay1.q_b = 0
    rc = sp.lib().sp_score_ex(FAKE, FAKE, C.byref(g1), C.byref(lay1), FAKE, FAKE, 1 << 20, _lib.SP_SCORE_SIMT, None)
    assert rc != _lib.SP_EINVAL


def test_seq_select_validation():
    """Sequence-sharded select: N divisible by the ranks, shards made of whole
    chunks, pooling half-window within one shard; M = min(K_c, n_c / P)."""
    L = sp.lib()
    p = _lib.sp_select_params(keep_rate=0.1, pool_k=5, chunk=32, pos0=0)
    assert L.sp_seq_candidate_count(131072, 8, C.byref(p)) == 410
    assert L.sp_seq_candidate_count(32768, 8, C.byref(p)) == 103
    p9 = _lib.sp_select_params(keep_rate=0.9, pool_k=5, chunk=32, pos0=0)
    assert L.sp_seq_candidate_count(131072, 8, C.byref(p9)) == 512          # keep >= 1/P: every chunk
    assert L.sp_seq_candidate_count(1000, 3, C.byref(p)) == -1                # N % P != 0
    assert L.sp_seq_candidate_count(3000, 3, C.byref(p)) == -1                # shard not whole chunks
    pw = _lib.sp_select_params(keep_rate=0.1, pool_k=41, chunk=1, pos0=0)
    assert L.sp_seq_candidate_count(128, 8, C.byref(pw)) == -1                # w = 20 > 16 tokens per shard
    assert L.sp_seq_select_workspace_bytes(1, 1000, 3, C.byref(p)) == 0
    assert L.sp_seq_select_workspace_bytes(2, 131072, 8, C.byref(p)) >= 2 * 4096 * 4
    assert L.sp_seq_candidates(FAKE, FAKE, 8, 8, 1, 131072, C.byref(p), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    assert L.sp_seq_merge(None, 8, 1, 131072, C.byref(p), None, FAKE, FAKE, FAKE, None, FAKE, 1 << 20, None) \
        == _lib.SP_EINVAL
    assert L.sp_seq_edges(FAKE, 1, 1000, 3, C.byref(p), FAKE, None) == _lib.SP_EINVAL


@pytest.mark.parametrize("keep,pool,chunk,code", [
    (0.0, 3, 4, _lib.SP_EINVAL), (1.01, 3, 4, _lib.SP_EINVAL), (float("nan"), 3, 4, _lib.SP_EINVAL),
    (0.5, 2, 4, _lib.SP_EINVAL), (0.5, 0, 4, _lib.SP_EINVAL), (0.5, 3, 0, _lib.SP_EINVAL),
])
def test_select_validation(keep, pool, chunk, code):
    p = _lib.sp_select_params(keep_rate=keep, pool_k=pool, chunk=chunk, pos0=0)
    rc = sp.lib().sp_select(FAKE, 1, 64, C.byref(p), FAKE, FAKE, FAKE, FAKE, 1 << 20, None)
    assert rc == code
    assert sp.lib().sp_select_workspace_bytes(1, 64, C.byref(p)) == 0


def test_gather_validation():
    assert sp.lib().sp_gather(None, FAKE, FAKE, 1, 10, FAKE, None) == _lib.SP_EINVAL
    assert sp.lib().sp_gather(FAKE, FAKE, FAKE, 0, 10, FAKE, None) == _lib.SP_EINVAL


def test_workspace_sizes_positive():
    g = _geom()
    assert sp.lib().sp_score_workspace_bytes(C.byref(g), _lib.SP_SCORE_SIMT) > 0
    assert sp.lib().sp_score_split_workspace_bytes(C.byref(g)) > 0
    p = _lib.sp_select_params(keep_rate=0.5, pool_k=3, chunk=4, pos0=0)
    assert sp.lib().sp_select_workspace_bytes(1, 64, C.byref(p)) >= 16 * 4


def test_no_cpu_fallback_without_device():
    """With valid arguments and no usable sm_100 device the call fails (it
    never computes on the CPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    g = _geom()
    lay = _layout(g)
    rc = sp.lib().sp_score(FAKE, FAKE, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 30, None)
    assert rc in (_lib.SP_ECUDA, _lib.SP_EUNSUPPORTED)


@pytest.mark.parametrize("name,variant", [("C0", {}), ("C1", {}), ("C2", {}), ("C3", {}), ("C4", {}),
                                          ("C3", dict(R=4)), ("C3", dict(H=32, Hkv=32, R=1)),
                                          ("C2", dict(B=200)), ("C1", dict(d=64)), ("C1", dict(d=256))])
def test_fused_plan_invariants(name, variant):
    """The fused kernel's host plan (no device needed: 148 SMs assumed): every
    request's jobs fit one wave of co-resident CTAs, a unit's tiles fit the
    TMEM ring, the SMEM carve fits the 227 KB limit."""
    import torch
    from spgen import gen
    w = gen.CONFIGS[name].with_(**variant)
    Q = torch.empty((w.B, w.L, w.R, w.H, w.d), dtype=torch.bfloat16, device="meta")
    K = torch.empty((w.B, w.L, w.Hkv, w.N, w.d), dtype=torch.bfloat16, device="meta")
    pl = sp.score_plan(Q, K, w.Rv)
    P, J = 148, pl["jobs_per_request"]
    T, U = -(-w.N // 128), w.L * w.Hkv
    assert pl["token_groups"] * pl["unit_groups"] == J
    assert pl["tiles_per_job"] == -(-T // pl["token_groups"]) and pl["units_per_job"] == -(-U // pl["unit_groups"])
    assert pl["grid"] == min(P, w.B * J)
    if w.B * J > P:
        assert P % J == 0                      # a request never straddles two waves
    assert pl["tiles_per_job"] <= pl["tmem_slots"]
    assert 2 <= pl["stages"] and pl["smem_bytes"] <= 232448
    assert pl["hier"] in (0, 1)


# ---------------------------------------------------------------- rows f3 / f4 host-side validation
def test_e4m3_validation():
    g = _geom(d=32)
    lay = _layout(g)
    e = sp.lib().sp_score_e4m3
    assert e(FAKE, FAKE, 0.0, 1.0, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    assert e(FAKE, FAKE, 1.0, float("inf"), C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    g16 = _geom(d=16)
    assert e(FAKE, FAKE, 1.0, 1.0, C.byref(g16), C.byref(_layout(g16)), FAKE, FAKE, 1 << 20, None) == \
        _lib.SP_EUNSUPPORTED                              # d % 32 != 0: no 32-byte swizzle rows
    lay.k_i = 40                                          # 40 B rows: not a multiple of 16 B
    assert e(FAKE, FAKE, 1.0, 1.0, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL


def _paged(g, **kw):
    pk = dict(cache=FAKE, s_l=64 * 16 * g.Hkv * g.d, s_blk=16 * g.Hkv * g.d, s_tok=g.Hkv * g.d, s_g=g.d,
              num_blocks=64, block_size=16, block_table=FAKE, max_blocks=-(-g.N // 16), seq_lens=None)
    pk.update(kw)
    return _lib.sp_paged_k(**pk)


@pytest.mark.parametrize("kw", [dict(block_size=4), dict(block_size=24), dict(block_size=384),
                                dict(max_blocks=1), dict(num_blocks=0), dict(cache=0), dict(block_table=0),
                                dict(s_tok=-8), dict(cache=FAKE + 8)])
def test_paged_validation(kw):
    g = _geom(d=64)
    pk = _paged(g, **kw)
    if "block_size" in kw:
        pk.max_blocks = 1 << 20
    rc = sp.lib().sp_score_paged(FAKE, C.byref(pk), C.byref(g), C.byref(_layout(g)), FAKE, FAKE, 1 << 20, None)
    assert rc == _lib.SP_EINVAL


def test_lookahead_and_ragged_validation():
    g = _geom()
    lay = _layout(g)
    la = _lib.sp_lookahead_k(K_la=FAKE, s_b=0, s_l=0, s_g=0, s_j=g.d, la_shift=2)
    f = sp.lib().sp_score_lookahead
    assert f(FAKE, FAKE, C.byref(la), C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    la.la_shift, la.s_j = 0, -1
    assert f(FAKE, FAKE, C.byref(la), C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    assert f(FAKE, FAKE, None, C.byref(g), C.byref(lay), FAKE, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    p = _lib.sp_select_params(keep_rate=0.5, pool_k=3, chunk=4, pos0=0)
    r = sp.lib().sp_select_ragged
    assert r(FAKE, None, None, 2, 100, C.byref(p), FAKE, FAKE, FAKE, None, FAKE, 1 << 20, None) == _lib.SP_EINVAL
    assert r(FAKE, FAKE, FAKE, 2, 100, C.byref(p), FAKE, FAKE, FAKE, None, FAKE, 1 << 20, None) == _lib.SP_EINVAL


@pytest.mark.parametrize("pool,chunk,cs,code", [
    (4, 32, FAKE, _lib.SP_EINVAL),          # even pool window
    (0, 32, FAKE, _lib.SP_EINVAL),
    (5, 0, FAKE, _lib.SP_EINVAL),           # empty chunk
    (5, 32, None, _lib.SP_EINVAL),          # no chunk-score output
    (4099, 32, FAKE, _lib.SP_EUNSUPPORTED),  # pool window above the staged halo
    (5, 16385, FAKE, _lib.SP_EUNSUPPORTED),  # chunk longer than a selection segment
])
def test_score_chunks_validation(pool, chunk, cs, code):
    """sp_score_chunks rejects bad selection parameters on the host (no device use)."""
    g = _geom()
    lay = _layout(g)
    rc = sp.lib().sp_score_chunks(FAKE, FAKE, C.byref(g), C.byref(lay), pool, chunk, FAKE, cs, FAKE, 1 << 20, None)
    assert rc == code
