"""Row f4: FP8 e4m3 Q/K through sp_score_e4m3 vs the float64 oracle.

The oracle decodes the same e4m3 codes itself (oracle.ref.e4m3_to_f64, pinned
in test_oracle.py) and runs the unchanged definition on the
dequantised values; parity bar as for bf16: importance within
1e-3 relative, ids/pos bit-exact beyond the 1e-3 margin, gathers bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import cuda as spgen_cuda
from spgen import fp8, gen
from tests import _util

pytestmark = pytest.mark.gpu

QS, KS = 1.0 / fp8.Q_INV_SCALE, 1.0 / fp8.K_INV_SCALE


def _bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)


def _codes_host(w: gen.Workload):
    """Host-generated bf16 inputs of every request, as e4m3 codes (numpy uint8)."""
    Qb, Kb, tok = gen.gen_batch(w)
    q8 = fp8.to_e4m3_codes(_bf16(Qb), fp8.Q_INV_SCALE).numpy()
    k8 = fp8.to_e4m3_codes(_bf16(Kb), fp8.K_INV_SCALE).numpy()
    return q8, k8, tok


def _oracle_imp(q8_b: np.ndarray, k8_b: np.ndarray, w: gen.Workload) -> np.ndarray:
    return ref.token_importance(QS * ref.e4m3_to_f64(q8_b), KS * ref.e4m3_to_f64(k8_b), w.scale, w.Rv)


def _small(w: gen.Workload, k_pad: int = 0):
    q8, k8, tok = _codes_host(w)
    Q = torch.from_numpy(q8).cuda()
    if k_pad:
        Kfull = torch.zeros((w.B, w.L, w.Hkv, w.N + k_pad, w.d), dtype=torch.uint8, device="cuda")
        Kfull[:, :, :, :w.N] = torch.from_numpy(k8).cuda()
        K = Kfull[:, :, :, :w.N]
    else:
        K = torch.from_numpy(k8).cuda()
    imp = sp.score_e4m3(Q, K, QS, KS, R_valid=w.Rv, scale=w.scale)
    sp.check_device_error()
    imp = imp.double().cpu().numpy()
    for b in range(w.B):
        err = _util.rel_err(imp[b], _oracle_imp(q8[b], k8[b], w))
        assert err <= _util.REL_TOL, f"{w} b={b}: importance rel err {err:.3e}"
    return q8, k8, tok, imp


@pytest.mark.parametrize("seed", range(3))
def test_e4m3_c0_d32(seed):
    _small(gen.CONFIGS["C0"].with_(d=32, seed=seed))


@pytest.mark.parametrize("variant", [
    dict(N=1), dict(N=5), dict(N=127), dict(N=129), dict(N=1000),
    dict(R=4, R_valid=2), dict(R=1), dict(R=9, N=300),
    dict(d=64), dict(d=96), dict(d=128), dict(d=256),
    dict(H=4, Hkv=4), dict(H=16, Hkv=2, R=4), dict(B=3, N=200), dict(L=5, N=333),
])
def test_e4m3_geometries(variant):
    w = gen.CONFIGS["C0"].with_(**{"d": 32, **variant})
    _small(w)


def test_e4m3_strided_cache():
    _small(gen.CONFIGS["C0"].with_(N=300, B=2, d=64), k_pad=48)


@pytest.mark.parametrize("plan,N", [("1,1", 2000), ("2,2", 4000), ("37,1", 5000), ("37,4", 5000)])
def test_e4m3_forced_plans(plan, N, monkeypatch):
    monkeypatch.setenv("SP_FUSED_PLAN", plan)
    w = gen.CONFIGS["C0"].with_(L=4, H=8, Hkv=2, d=128, N=N, R=3, B=2)
    q8, k8, _ = _codes_host(w)
    pl = sp.score_e4m3_plan(torch.from_numpy(q8).cuda(), torch.empty((w.B, w.L, w.Hkv, w.N, w.d), dtype=torch.uint8,
                                                                     device="cuda"))
    assert (pl["token_groups"], pl["unit_groups"]) == tuple(int(x) for x in plan.split(","))
    _small(w)


def test_e4m3_d16_unsupported():
    w = gen.CONFIGS["C0"]
    q8, k8, _ = _codes_host(w)
    with pytest.raises(sp.SpError) as e:
        sp.score_e4m3(torch.from_numpy(q8).cuda(), torch.from_numpy(k8).cuda(), QS, KS, scale=w.scale)
    assert e.value.code == 2


def test_e4m3_matches_bf16_kernel_on_dequantised_values():
    """The e4m3 kernel and the bf16 kernel on the dequantised values (exact in
    bf16: e4m3 has 4 significant bits) give the same importance to fp32 rounding."""
    w = gen.CONFIGS["C1"].with_(N=1500)
    q8, k8, _ = _codes_host(w)
    Qd = torch.from_numpy(QS * ref.e4m3_to_f64(q8)).to(torch.bfloat16).cuda()
    Kd = torch.from_numpy(KS * ref.e4m3_to_f64(k8)).to(torch.bfloat16).cuda()
    a = sp.score_e4m3(torch.from_numpy(q8).cuda(), torch.from_numpy(k8).cuda(), QS, KS, R_valid=w.Rv, scale=w.scale)
    b = sp.score(Qd, Kd, R_valid=w.Rv, scale=w.scale, algo="fused")
    sp.check_device_error()
    assert _util.rel_err(a.double().cpu().numpy(), b.double().cpu().numpy()) <= 1e-5


def _full(w: gen.Workload, requests):
    Q, K, T = spgen_cuda.make_inputs(w)
    Q8 = fp8.to_e4m3_codes(Q, fp8.Q_INV_SCALE)
    K8 = fp8.to_e4m3_codes(K, fp8.K_INV_SCALE)
    del K
    imp = sp.score_e4m3(Q8, K8, QS, KS, R_valid=w.Rv, scale=w.scale)
    ids, pos, nk = sp.select(imp, w.keep, w.pool_k, w.chunk, w.pos0)
    out = sp.gather(T, ids, nk)
    sp.check_device_error()
    a = sp.score_e4m3(Q8, K8, QS, KS, R_valid=w.Rv, scale=w.scale)
    assert torch.equal(a, imp), "not deterministic"
    for b in requests:
        q8 = Q8[b].cpu().numpy()
        Qf = QS * ref.e4m3_to_f64(q8)
        exact = ref.token_importance(Qf, lambda l: KS * ref.e4m3_to_f64(K8[b, l].cpu().numpy()), w.scale, w.Rv)
        err = _util.rel_err(imp[b].double().cpu().numpy(), exact)
        assert err <= _util.REL_TOL, f"b={b}: importance rel err {err:.3e}"
        o = ref.select(exact, w.keep, w.pool_k, w.chunk, w.pos0)
        n = int(nk[b])
        _util.check_selection(ids[b].cpu().numpy(), pos[b].cpu().numpy(), n, o, w.chunk, w.N, w.pos0)
        assert torch.equal(out[b, :n], T[b][ids[b, :n].long()])


def test_e4m3_c1_full():
    _full(gen.CONFIGS["C1"], [0])


def test_e4m3_c2_sampled():
    _full(gen.CONFIGS["C2"], [0, 40])


def test_e4m3_c3_full():
    _full(gen.CONFIGS["C3"], [0])
