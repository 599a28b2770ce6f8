"""Row f4, reading Z2': the look-ahead tokens' keys in
each row's softmax denominator, sp_score_lookahead vs the float64 oracle
(oracle.ref.attention_scores_lookahead, pinned in test_oracle.py)."""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import gen
from tests import _util

pytestmark = pytest.mark.gpu


def _dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _case(w: gen.Workload, shift: int, tol=_util.REL_TOL):
    Qb, Kb, _ = gen.gen_batch(w)
    wl = w.with_(N=w.R, seed=w.seed + 1000)                      # look-ahead keys: R rows per (b, l, g)
    Klb = np.stack([np.stack([np.stack([gen.gen_K(wl, b, l, g) for g in range(w.Hkv)]) for l in range(w.L)])
                    for b in range(w.B)])
    imp = sp.score_lookahead(_dev(Qb), _dev(Kb), _dev(Klb), shift, R_valid=w.Rv, scale=w.scale)
    sp.check_device_error()
    imp = imp.double().cpu().numpy()
    for b in range(w.B):
        A = ref.attention_scores_lookahead(ref.bf16_to_f64(Qb[b])[:, :w.Rv], ref.bf16_to_f64(Kb[b]),
                                           ref.bf16_to_f64(Klb[b]), w.scale, shift)
        exact = ref.aggregate_attention(A)
        err = _util.rel_err(imp[b], exact)
        assert err <= tol, f"{w} shift={shift} b={b}: rel err {err:.3e}"
    return imp


@pytest.mark.parametrize("shift", [0, 1])
@pytest.mark.parametrize("variant", [
    dict(), dict(N=5), dict(N=129), dict(N=1000), dict(R=4, R_valid=2), dict(R=1), dict(R=9, N=300),
    dict(d=64), dict(d=128), dict(H=16, Hkv=2, R=4), dict(B=3, N=200), dict(L=5, N=333),
])
def test_lookahead_geometries(variant, shift):
    _case(gen.CONFIGS["C0"].with_(**variant), shift)


def test_lookahead_strong_keys_lower_importance():
    """Look-ahead keys aligned with the queries take probability mass from the
    prompt: importance strictly below the prompt-only reading (same inputs)."""
    w = gen.CONFIGS["C0"].with_(N=300, R=4, d=64)
    Qb, Kb, _ = gen.gen_batch(w)
    Q = _dev(Qb)
    Kla = Q.permute(0, 1, 3, 2, 4)[:, :, ::w.G].contiguous() * 4        # k_la[j] = 4 * q[r=j] of head g*G
    a = sp.score_lookahead(Q, _dev(Kb), Kla, 0, scale=w.scale)
    b = sp.score(Q, _dev(Kb), scale=w.scale, algo="fused")
    assert (a < b).all()


def test_lookahead_8b_geometry():
    """8B head geometry (L32 H32 Hkv8 d128 R8) at a short prompt, both shifts."""
    w = gen.CONFIGS["C1"].with_(N=600, seed=3)
    for shift in (0, 1):
        _case(w, shift)
