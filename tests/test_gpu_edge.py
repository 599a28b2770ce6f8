"""Edge cases of the fused path vs the float64 oracle: batches that
need several waves of CTAs, single-token prompts at the 8B geometry, peaked and
flat softmaxes, and the extreme keep rates."""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import cuda as spgen_cuda
from spgen import gen
from tests import _util

pytestmark = pytest.mark.gpu


def _dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("B,N", [(300, 37), (160, 300), (149, 1)])
def test_multi_wave_batches(B, N):
    """More jobs than SMs: requests are scheduled in several waves of the
    persistent grid (a request never straddles two waves)."""
    w = gen.CONFIGS["C1"].with_(B=B, N=N, L=4, seed=7)
    Q, K, T = spgen_cuda.make_inputs(w)
    plan = sp.score_plan(Q, K, w.Rv)
    assert B * plan["jobs_per_request"] > plan["grid"]
    imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    ids, pos, nk = sp.select(imp, w.keep, w.pool_k, w.chunk)
    sp.check_device_error()
    for b in (0, B // 2, B - 1):
        exact = _util.oracle_importance(w, b)
        assert _util.rel_err(imp[b].double().cpu().numpy(), exact) <= _util.REL_TOL, b
        o = ref.select(exact, w.keep, w.pool_k, w.chunk)
        _util.check_selection(ids[b].cpu().numpy(), pos[b].cpu().numpy(), int(nk[b]), o, w.chunk, N, 0)


def test_single_token_8b():
    """N = 1: every probability is 1, importance exactly 1."""
    w = gen.CONFIGS["C1"].with_(N=1)
    Q, K, T = spgen_cuda.make_inputs(w)
    imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    sp.check_device_error()
    assert torch.allclose(imp, torch.ones_like(imp), rtol=1e-6, atol=0)


@pytest.mark.parametrize("scale", [4.0, 1e-3])
def test_peaked_and_flat_softmax(scale):
    """A large scale (peaked rows: probabilities spanning hundreds of binades,
    the running-reference re-base path) and a tiny one (nearly uniform rows)."""
    w = gen.CONFIGS["C0"].with_(N=700, d=64, R=3)
    Qb, Kb, _ = gen.gen_batch(w)
    imp = sp.score(_dev(Qb), _dev(Kb), scale=scale, algo="fused")
    sp.check_device_error()
    exact = ref.token_importance(ref.bf16_to_f64(Qb[0]), ref.bf16_to_f64(Kb[0]), float(np.float32(scale)))
    got = imp[0].double().cpu().numpy()
    big = exact > 1e-30                       # below ~2^-100 both sides flush to zero (ex2.approx.ftz)
    assert _util.rel_err(got[big], exact[big]) <= _util.REL_TOL
    assert np.all(got[~big] <= 1e-30)


@pytest.mark.parametrize("keep", [1e-6, 1.0])
def test_extreme_keep_rates(keep):
    w = gen.CONFIGS["C1"].with_(N=3000)
    Q, K, T = spgen_cuda.make_inputs(w)
    imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    ids, pos, nk, out = sp.select(imp, keep, w.pool_k, w.chunk, pos0=5, tokens=T)
    sp.check_device_error()
    exact = _util.oracle_importance(w, 0)
    o = ref.select(exact, keep, w.pool_k, w.chunk, 5)
    n = int(nk[0])
    _util.check_selection(ids[0].cpu().numpy(), pos[0].cpu().numpy(), n, o, w.chunk, w.N, 5)
    assert n == (w.chunk if keep < 1 else w.N)
    assert torch.equal(out[0, :n], T[0][ids[0, :n].long()])
