"""Row f3: paged K cache (block table) and ragged batches vs the oracle.

The same seeded keys are laid out in a vLLM-style paged cache
[L][num_blocks][block_size][Hkv][d] with a shuffled block table; the oracle
scores each request over its own n_b prompt tokens (softmax over
the prompt keys, Z2) and selects over them.  Parity bar as for the
contiguous path.
"""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import cuda as spgen_cuda
from spgen import gen, paged
from tests import _util

pytestmark = pytest.mark.gpu


def _paged(K: torch.Tensor, bs: int, seed: int = 0, spare: int = 3, layout: str = "nhd"):
    return paged.to_paged(K, bs, seed, spare, layout)


def _oracle_req(Qb, Kb, w, n):
    return ref.token_importance(ref.bf16_to_f64(Qb), ref.bf16_to_f64(Kb[:, :, :n]), w.scale, w.Rv)


def _dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("layout", ["nhd", "hnd"])
@pytest.mark.parametrize("bs", [8, 16, 32, 64, 128, 256])
def test_paged_uniform_bitexact_vs_contiguous(bs, layout, d):
    """Paging only changes where the TMA reads a tile from (d >= 128 with blocks
    < 128 tokens: one box per block, kb halves interleaved per 8-row group): the
    importance is bit-identical to sp_score on the contiguous cache, and within
    1e-3 of the oracle."""
    w = gen.CONFIGS["C0"].with_(L=3, H=8, Hkv=2, d=d, R=3, N=1000, B=2)
    Qb, Kb, _ = gen.gen_batch(w)
    Q, K = _dev(Qb), _dev(Kb)
    cache, bt = _paged(K, bs, seed=bs, layout=layout)
    imp = sp.score_paged(Q, cache, bt, N=w.N, R_valid=w.Rv, scale=w.scale)
    ref_imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    sp.check_device_error()
    assert torch.equal(imp, ref_imp)
    for b in range(w.B):
        assert _util.rel_err(imp[b].double().cpu().numpy(), _oracle_req(Qb[b], Kb[b], w, w.N)) <= _util.REL_TOL


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bs", [16, 128])
@pytest.mark.parametrize("lens", [(1000, 337, 77), (64, 1, 129), (5000, 4999, 128, 2500)])
def test_ragged_paged_vs_oracle(bs, lens, d):
    """Requests of different lengths in one launch: each request's softmax runs
    over its own prompt keys; the selection over its own chunks."""
    N = max(lens)
    w = gen.CONFIGS["C0"].with_(L=2, H=8, Hkv=2, d=d, R=3, N=N, B=len(lens), keep=0.3, pool_k=5, chunk=8)
    Qb, Kb, tok = gen.gen_batch(w)
    Q, K = _dev(Qb), _dev(Kb)
    cache, bt = _paged(K, bs)
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    imp = sp.score_paged(Q, cache, bt, seq, N=N, R_valid=w.Rv, scale=w.scale)
    T = torch.tensor(tok, dtype=torch.int32, device="cuda")
    ids, pos, nk, out = sp.select_ragged(imp, seq, w.keep, w.pool_k, w.chunk, pos0=3, tokens=T)
    sp.check_device_error()
    for b, n in enumerate(lens):
        exact = _oracle_req(Qb[b], Kb[b], w, n)
        assert _util.rel_err(imp[b, :n].double().cpu().numpy(), exact) <= _util.REL_TOL, (b, n)
        o = ref.select(exact, w.keep, w.pool_k, w.chunk, 3)
        k = int(nk[b])
        _util.check_selection(ids[b].cpu().numpy(), pos[b].cpu().numpy(), k, o, w.chunk, n, 3)
        assert torch.equal(out[b, :k], T[b][ids[b, :k].long()])


def test_ragged_select_dyadic_ties_bitexact():
    """Exact fp32 sums: the per-request tie-break and K_c match the oracle bit for bit."""
    rng = np.random.default_rng(3)
    B, N = 5, 9000
    imp = rng.integers(0, 4, size=(B, N)).astype(np.float64) / 64.0
    lens = [9000, 1, 31, 4097, 8191]
    for chunk, keep in [(8, 0.25), (1, 0.1), (32, 0.9)]:
        seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
        ids, pos, nk = sp.select_ragged(torch.tensor(imp, dtype=torch.float32, device="cuda"), seq, keep, 1, chunk)
        for b, n in enumerate(lens):
            o = ref.select(imp[b, :n], keep, 1, chunk, 0)
            k = int(nk[b])
            assert k == o["n_kept"], (chunk, b)
            np.testing.assert_array_equal(ids[b, :k].cpu().numpy(), o["ids"])


def test_ragged_select_uniform_equals_select():
    rng = np.random.default_rng(4)
    imp = torch.tensor(rng.random((3, 50000)) ** 4 + 1e-6, dtype=torch.float32, device="cuda")
    seq = torch.full((3,), 50000, dtype=torch.int32, device="cuda")
    a = sp.select(imp, 0.1, 5, 32, pos0=2)
    b = sp.select_ragged(imp, seq, 0.1, 5, 32, pos0=2)
    assert torch.equal(a[2], b[2])
    for r in range(3):
        n = int(a[2][r])
        assert torch.equal(a[0][r, :n], b[0][r, :n]) and torch.equal(a[1][r, :n], b[1][r, :n])


def test_paged_invalid_block_size():
    w = gen.CONFIGS["C0"].with_(d=64, N=100)
    Qb, Kb, _ = gen.gen_batch(w)
    Q, K = _dev(Qb), _dev(Kb)
    for bs in (4, 24, 192, 384):
        cache = torch.zeros((w.L, 64, bs, w.Hkv, w.d), dtype=torch.bfloat16, device="cuda")
        bt = torch.zeros((1, -(-w.N // bs)), dtype=torch.int32, device="cuda")
        with pytest.raises(sp.SpError) as e:
            sp.score_paged(Q, cache, bt, N=w.N, scale=w.scale)
        assert e.value.code == 1


@pytest.mark.parametrize("layout", ["nhd", "hnd"])
def test_paged_c1_full_bitexact(layout):
    """8B geometry, 4K prompt, vLLM's default block size 16: bit-identical to the contiguous path."""
    w = gen.CONFIGS["C1"]
    Q, K, T = spgen_cuda.make_inputs(w)
    cache, bt = _paged(K, 16, layout=layout)
    imp = sp.score_paged(Q, cache, bt, N=w.N, R_valid=w.Rv, scale=w.scale)
    ref_imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    sp.check_device_error()
    assert torch.equal(imp, ref_imp)


def test_paged_ragged_c2_sampled():
    """C2-shaped batch (64 requests, 8B geometry) with ragged lengths in a
    block-16 paged cache; the oracle checks a sample of requests."""
    w = gen.CONFIGS["C2"]
    Q, K, T = spgen_cuda.make_inputs(w)
    rng = np.random.default_rng(9)
    lens = rng.integers(200, w.N + 1, size=w.B)
    lens[0], lens[17] = w.N, 1
    cache, bt = _paged(K, 16, layout="hnd")
    del K
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    imp = sp.score_paged(Q, cache, bt, seq, N=w.N, R_valid=w.Rv, scale=w.scale)
    ids, pos, nk = sp.select_ragged(imp, seq, w.keep, w.pool_k, w.chunk)
    sp.check_device_error()
    for b in (0, 17, 40):
        n = int(lens[b])
        Qf = ref.bf16_to_f64(np.stack([gen.gen_Q(w, b, l) for l in range(w.L)]))
        exact = ref.token_importance(Qf, lambda l: _util.k_layer_f64(w, b, l, 0, n), w.scale, w.Rv)
        assert _util.rel_err(imp[b, :n].double().cpu().numpy(), exact) <= _util.REL_TOL, b
        o = ref.select(exact, w.keep, w.pool_k, w.chunk)
        _util.check_selection(ids[b].cpu().numpy(), pos[b].cpu().numpy(), int(nk[b]), o, w.chunk, n, 0)


@pytest.mark.parametrize("d,bs", [(128, 16), (128, 128), (256, 16), (64, 32)])
def test_paged_e4m3_bitexact_vs_contiguous(d, bs):
    """Rows f3 x f4: an FP8 paged cache gives the e4m3 contiguous path's bits."""
    from spgen import fp8
    w = gen.CONFIGS["C0"].with_(L=3, H=8, Hkv=2, d=d, R=3, N=1000, B=2)
    Qb, Kb, _ = gen.gen_batch(w)
    Q8, K8 = fp8.to_e4m3_codes(_dev(Qb), fp8.Q_INV_SCALE), fp8.to_e4m3_codes(_dev(Kb), fp8.K_INV_SCALE)
    qs, ks = 1 / fp8.Q_INV_SCALE, 1 / fp8.K_INV_SCALE
    cache, bt = _paged(K8, bs, layout="hnd")
    a = sp.score_paged(Q8, cache, bt, N=w.N, R_valid=w.Rv, scale=w.scale, q_scale=qs, k_scale=ks)
    b = sp.score_e4m3(Q8, K8, qs, ks, R_valid=w.Rv, scale=w.scale)
    sp.check_device_error()
    assert torch.equal(a, b)
    exact = ref.token_importance(qs * ref.e4m3_to_f64(Q8[0].cpu().numpy()), ks * ref.e4m3_to_f64(K8[0].cpu().numpy()),
                                 w.scale, w.Rv)
    assert _util.rel_err(a[0].double().cpu().numpy(), exact) <= _util.REL_TOL
