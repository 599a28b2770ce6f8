"""sp_score_select (the score kernel computes the selection's chunk scores in its
epilogue, the dependent selection launch runs phases B-C; or, where the epilogue
cannot stage them, the score then the whole selection) gives exactly sp_score +
sp_select_gather's outputs, over the score kernel's decompositions (one or
several unit groups per token group, several waves of CTAs), chunk sizes that
do not divide a tile, pooling halos reaching across token groups, repeated
calls (the ready tags and counters run across launches) and B > 1."""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import cuda as spgen_cuda
from spgen import gen
from tests import _util

pytestmark = pytest.mark.gpu


def _both(w, keep=None, pool_k=None, chunk=None, pos0=0, reps=3):
    keep = w.keep if keep is None else keep
    pool_k = w.pool_k if pool_k is None else pool_k
    chunk = w.chunk if chunk is None else chunk
    Q, K, T = spgen_cuda.make_inputs(w)
    imp0 = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="auto")
    ids0, pos0_, nk0, out0 = sp.select(imp0, keep, pool_k, chunk, pos0, tokens=T)
    for _ in range(reps):
        imp, ids, pos, nk, out = sp.score_select(Q, K, keep, pool_k, chunk, pos0, tokens=T, R_valid=w.Rv,
                                                 scale=w.scale)
        sp.check_device_error()
        assert torch.equal(imp, imp0)
        assert torch.equal(nk, nk0)
        for b in range(w.B):
            n = int(nk0[b])
            assert torch.equal(ids[b, :n], ids0[b, :n]) and torch.equal(pos[b, :n], pos0_[b, :n])
            assert torch.equal(out[b, :n], out0[b, :n])
    return imp, ids, pos, nk, out, T


@pytest.mark.parametrize("name,kw,sel", [
    ("C0", {}, {}),
    ("C1", {}, {}),                                  # one CTA runs the selection (2 chunk blocks)
    ("C3", {}, {}),                                  # phase A over 16 CTAs
    ("C1", dict(N=9000), dict(chunk=1, pool_k=5)),   # token-level chunks, partial tail block
    ("C1", dict(N=20000, L=4), dict(chunk=24, pool_k=33)),
    ("C1", dict(N=5000, R_valid=5), dict(chunk=100, pool_k=1, pos0=7)),
    ("C1", dict(B=2, N=3000), {}),                   # B > 1
    ("C2", dict(B=8), {}),                           # medium prompts, several requests per wave
    ("C1", dict(B=160, N=256, L=2), dict(chunk=8, pool_k=9)),        # several waves of the persistent grid
    ("C1", dict(N=6000, L=2), dict(chunk=32, pool_k=1025)),          # halo over several token groups (or fallback)
    ("C1", dict(N=7777, L=4), dict(chunk=48, pool_k=65, pos0=3)),    # chunks straddling token groups
    ("C1", dict(N=4096, L=4, R_valid=1), {}),                        # R = 1: the epilogue cannot stage (fallback)
])
def test_score_select_equals_two_launches(name, kw, sel):
    _both(gen.CONFIGS[name].with_(**kw), **sel)


@pytest.mark.parametrize("plan", ["148,1", "37,4", "8,16", "64,2"])
def test_score_select_forced_plans(plan, monkeypatch):
    """Every epilogue decomposition: one CTA per token group (n_ug = 1) or several."""
    monkeypatch.setenv("SP_FUSED_PLAN", plan)
    _both(gen.CONFIGS["C3"].with_(N=16384, L=8), reps=2)


@pytest.mark.slow
def test_score_select_c4_keep_sweep():
    """C4 (phase A over 64 CTAs of the 138-CTA grid), each keep rate twice."""
    w = gen.CONFIGS["C4"]
    Q, K, T = spgen_cuda.make_inputs(w)
    imp0 = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    for k in (1, 5, 9):
        keep = k / 10.0
        ids0, pos0, nk0, out0 = sp.select(imp0, keep, w.pool_k, w.chunk, tokens=T)
        for _ in range(2):
            imp, ids, pos, nk, out = sp.score_select(Q, K, keep, w.pool_k, w.chunk, tokens=T, R_valid=w.Rv,
                                                     scale=w.scale)
            sp.check_device_error()
            n = int(nk0[0])
            assert torch.equal(imp, imp0) and int(nk[0]) == n
            assert torch.equal(ids[0, :n], ids0[0, :n]) and torch.equal(out[0, :n], out0[0, :n])


def test_score_select_planted_c3_vs_oracle():
    """The fused call on the planted 32K fixture selects the oracle's ids bit-exactly."""
    w = gen.CONFIGS["C3"].with_(planted=True)
    imp, ids, pos, nk, out, T = _both(w, reps=1)
    exact = _util.oracle_importance(w, 0)
    o = ref.select(exact, w.keep, w.pool_k, w.chunk)
    reg = _util.check_selection(ids[0].cpu().numpy(), pos[0].cpu().numpy(), int(nk[0]), o, w.chunk, w.N, 0)
    _util.record(w, w.keep, 0, reg, ref.margin(o["cs"], o["K_c"]), _util.rel_err(imp[0].double().cpu().numpy(), exact),
                 "score_select")
    assert reg == "exact"
    n = int(nk[0])
    np.testing.assert_array_equal(out[0, :n].cpu().numpy(), T[0, ids[0, :n].long()].cpu().numpy())


@pytest.mark.parametrize("name,kw,sel", [
    ("C1", {}, {}),
    ("C3", dict(N=10000, L=4), dict(chunk=24, pool_k=33)),
    ("C1", dict(N=3001, L=2), dict(chunk=1, pool_k=7)),
])
def test_score_chunks_vs_oracle(name, kw, sel):
    """sp_score_chunks' chunk scores equal the oracle's pooling + chunk means
    (O5-O6) of the kernel's own importance, to fp32 summation rounding, and its
    importance equals sp_score's bit for bit."""
    w = gen.CONFIGS[name].with_(**kw)
    pool_k = sel.get("pool_k", w.pool_k)
    chunk = sel.get("chunk", w.chunk)
    Q, K, T = spgen_cuda.make_inputs(w)
    imp0 = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    imp, cs = sp.score_chunks(Q, K, pool_k, chunk, R_valid=w.Rv, scale=w.scale)
    sp.check_device_error()
    assert torch.equal(imp, imp0)
    x = imp[0].double().cpu().numpy()
    want = ref.chunk_scores(ref.smooth_scores(x, pool_k), chunk)
    got = cs[0].double().cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)


@pytest.mark.parametrize("name,kw,sel", [
    ("C1", {}, {}),
    ("C3", dict(N=16384, L=8), {}),
    ("C1", dict(N=7777, L=4), dict(chunk=48, pool_k=65, pos0=3)),
])
def test_score_select_epilogue_variant(name, kw, sel, monkeypatch):
    """The measured alternative (SP_SELECT_EPILOGUE): the chunk means in the score
    kernel's epilogue and a top-K_c-only selection launch -- the same bits."""
    monkeypatch.setenv("SP_SELECT_EPILOGUE", "1")
    _both(gen.CONFIGS[name].with_(**kw), reps=2, **sel)
