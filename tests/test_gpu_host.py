"""sp_run_host -- the call behind bench.py's e2e number: the whole path from
pinned host buffers (H2D, score, select + gather, D2H) against the float64
oracle, and bit-identical to the device-resident path."""
import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import gen
from tests import _util

pytestmark = pytest.mark.gpu


def _host_run(w):
    Qb, Kb, tok = gen.gen_batch(w)
    Qh = torch.from_numpy(Qb.view(np.int16)).view(torch.bfloat16).pin_memory()
    Kh = torch.from_numpy(Kb.view(np.int16)).view(torch.bfloat16).pin_memory()
    Th = torch.from_numpy(tok).pin_memory()
    dev = torch.device("cuda")
    ho = {k: torch.full((w.B, w.N), -1, dtype=torch.int32).pin_memory() for k in ("ids", "pos", "out_tokens")}
    ho["n_kept"] = torch.zeros((w.B,), dtype=torch.int32).pin_memory()
    Qd, Kd, Td = torch.empty_like(Qh, device=dev), torch.empty_like(Kh, device=dev), torch.empty_like(Th, device=dev)
    nbytes = sp.run_workspace_bytes(Qd, Kd, w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0)
    dv = {"Q": Qd, "K": Kd, "tokens": Td, "importance": torch.empty((w.B, w.N), dtype=torch.float32, device=dev),
          "ids": torch.empty_like(Td), "pos": torch.empty_like(Td),
          "n_kept": torch.empty((w.B,), dtype=torch.int32, device=dev), "out_tokens": torch.empty_like(Td),
          "ws": torch.zeros(nbytes, dtype=torch.uint8, device=dev)}
    for _ in range(2):                                   # the second call reuses the workspace (epoch, counters)
        sp.run_host(Qh, Kh, Th, dv, w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0, host_out=ho)
        torch.cuda.synchronize()
    sp.check_device_error()
    return Qb, Kb, tok, ho, dv


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C0", dict(pos0=9)), ("C1", dict(B=3, N=1500, R_valid=5, pos0=4))])
def test_run_host_vs_oracle(name, kw):
    w = gen.CONFIGS[name].with_(**kw)
    Qb, Kb, tok, ho, dv = _host_run(w)
    for b in range(w.B):
        o = ref.specprefill(Qb[b], Kb[b], tok[b], w.scale, w.keep, w.pool_k, w.chunk, w.Rv, w.pos0)
        n = int(ho["n_kept"][b])
        err = _util.rel_err(dv["importance"][b].double().cpu().numpy(), o["imp"])
        assert err <= _util.REL_TOL
        reg = _util.check_selection(ho["ids"][b].numpy(), ho["pos"][b].numpy(), n, o, w.chunk, w.N, w.pos0)
        _util.record(w, w.keep, b, reg, ref.margin(o["cs"], o["K_c"]), err, "run_host")
        ids = ho["ids"][b, :n].numpy()
        np.testing.assert_array_equal(ho["out_tokens"][b, :n].numpy(), tok[b][ids])      # gather: bit-exact
        # equal to the device-resident path on the same inputs
        Q = torch.from_numpy(Qb.view(np.int16)).view(torch.bfloat16).cuda()
        K = torch.from_numpy(Kb.view(np.int16)).view(torch.bfloat16).cuda()
        r = sp.specprefill(Q, K, torch.from_numpy(tok).cuda(), w.keep, w.pool_k, w.chunk, w.Rv, w.scale, w.pos0)
        assert int(r["n_kept"][b]) == n
        np.testing.assert_array_equal(r["ids"][b, :n].cpu().numpy(), ids)
        np.testing.assert_array_equal(r["pos"][b, :n].cpu().numpy(), ho["pos"][b, :n].numpy())
