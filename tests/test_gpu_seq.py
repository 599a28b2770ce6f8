"""Row e on the GPU: the sequence-sharded selection (sp_seq_edges ->
all-gather -> sp_seq_candidates -> all-gather -> sp_seq_merge) run as P
virtual ranks on one GPU (the all-gathers are torch.stack of the ranks'
buffers), bit-identical to sp_select_gather on the concatenated importance;
and the whole sequence-sharded path through torch.distributed (NCCL, symmetric
memory rendezvous) on a single-rank group."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2502_02789_b200 as sp
from oracle import ref
from spgen import cuda as spgen_cuda
from spgen import gen
from tests import _util

pytestmark = pytest.mark.gpu


def _virtual_ranks(imp, P, keep, pool_k, chunk, pos0, tokens):
    B, N = imp.shape
    n = N // P
    shards = [imp[:, p * n:(p + 1) * n].contiguous() for p in range(P)]
    edges = torch.stack([sp.seq_edges(shards[p], P, N, keep, pool_k, chunk) for p in range(P)]).contiguous()
    cand = torch.stack([sp.seq_candidates(shards[p], edges, p, P, N, keep, pool_k, chunk) for p in range(P)])
    M = sp.seq_candidate_count(N, P, keep, pool_k, chunk)
    assert tuple(cand.shape) == (P, B, M)
    return sp.seq_merge(cand.contiguous(), P, N, keep, pool_k, chunk, pos0, tokens=tokens)


def _check_equal(imp, P, keep, pool_k, chunk, pos0, tokens):
    a = _virtual_ranks(imp, P, keep, pool_k, chunk, pos0, tokens)
    b = sp.select(imp, keep, pool_k, chunk, pos0, tokens=tokens)
    sp.check_device_error()
    assert torch.equal(a[2], b[2]), (P, keep, pool_k, chunk, a[2], b[2])
    for r in range(imp.shape[0]):
        n = int(b[2][r])
        for x, y in zip(a[:2] + a[3:], b[:2] + b[3:]):
            assert torch.equal(x[r, :n], y[r, :n]), (P, keep, pool_k, chunk)
    return b


@pytest.fixture(scope="module")
def c4_importance():
    """The fused kernel's importance of the C4 prompt (default generator)."""
    w = gen.CONFIGS["C4"]
    Q, K, T = spgen_cuda.make_inputs(w)
    imp = sp.score(Q, K, R_valid=w.Rv, scale=w.scale, algo="fused")
    sp.check_device_error()
    del Q, K
    torch.cuda.empty_cache()
    return w, imp, T


@pytest.mark.parametrize("P", [2, 4, 8])
def test_seq_select_c4_keep_sweep(c4_importance, P):
    """C4 geometry (128K tokens, chunk 32, pool 5), keep 0.1..0.9 (keep >= 1/P
    degenerates into gathering every chunk score): bit-identical to the
    single-GPU selection."""
    w, imp, T = c4_importance
    for k in range(1, 10):
        _check_equal(imp, P, k / 10.0, w.pool_k, w.chunk, 0, T)


def test_seq_select_c4_vs_oracle(c4_importance):
    """The merged selection at P = 8 satisfies the oracle parity rule (the
    oracle's importance recomputed on the host for the C4 prompt)."""
    w, imp, T = c4_importance
    exact = _util.oracle_importance(w, 0)
    for keep in (0.1, 0.5, 0.9):
        ids, pos, nk, out = _virtual_ranks(imp, 8, keep, w.pool_k, w.chunk, 0, T)
        o = ref.select(exact, keep, w.pool_k, w.chunk, 0)
        n = int(nk[0])
        reg = _util.check_selection(ids[0].cpu().numpy(), pos[0].cpu().numpy(), n, o, w.chunk, w.N, 0)
        _util.record(w, keep, 0, reg, ref.margin(o["cs"], o["K_c"]),
                     _util.rel_err(imp[0].double().cpu().numpy(), exact), "seq_select_P8")
        assert torch.equal(out[0, :n], T[0][ids[0, :n].long()])


@pytest.mark.parametrize("chunk,pool_k", [(32, 5), (1, 1), (1, 3), (24, 9), (100, 33), (2048, 5), (17, 4097)])
@pytest.mark.parametrize("P", [2, 8])
def test_seq_select_cross_rank_ties(P, chunk, pool_k):
    """Importance whose chunk pattern repeats on every rank (identical local
    windows give identical fp32 chunk scores, so chunks tie across ranks; the
    lowest index must win), dyadic near-ties, several keep rates incl. >= 1/P,
    B = 2, pos0 > 0."""
    n = max(chunk * 64, (pool_k // 2 + 1) * 2)
    n = -(-n // chunk) * chunk
    N = n * P
    g = torch.Generator().manual_seed(chunk * 131 + pool_k)
    lev = torch.randint(1, 9, (2, n // chunk), generator=g).float() / 8.0
    pattern = lev.repeat_interleave(chunk, dim=1)                                  # [2][n]
    noise = torch.randint(0, 4, (2, n), generator=g).float() / 64.0
    imp = (pattern + noise).repeat(1, P).contiguous().cuda()                          # same pattern on every rank
    tok = torch.randint(0, 128256, (2, N), generator=g, dtype=torch.int32).cuda()
    for keep in (0.05, 1.0 / P, 0.5, 0.97):
        _check_equal(imp, P, keep, pool_k, chunk, 7, tok)


def test_seq_select_validation():
    imp = torch.rand((1, 1000), device="cuda")
    with pytest.raises(sp.SpError):
        sp.seq_edges(imp, 3, 3000, 0.1, 5, 32)        # shard not a multiple of chunk
    with pytest.raises(sp.SpError):
        sp.seq_candidate_count(3000, 3, 0.1, 4, 1)    # even pool_k
    with pytest.raises(sp.SpError):
        sp.seq_candidate_count(64, 8, 0.1, 21, 1)     # half-window wider than a shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(port, name, mode, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        from paper_2502_02789_b200 import dist as spd
        w = gen.CONFIGS[name].with_(N=8192, R_valid=6) if name != "C0" else gen.CONFIGS["C0"]
        Q, K, T = spgen_cuda.make_inputs(w)
        if mode == "fused":
            r = spd.seq_sharded_fused_specprefill(Q, K, T, w.N, w.keep, w.pool_k, w.chunk, w.Rv, w.scale)
            r2 = spd.seq_sharded_fused_specprefill(Q, K, T, w.N, w.keep, w.pool_k, w.chunk, w.Rv, w.scale)
            assert torch.equal(r["importance_local"], r2["importance_local"])
        else:
            r = spd.seq_sharded_specprefill(Q, K, T, w.N, w.keep, w.pool_k, w.chunk, w.Rv, w.scale)
        sp.check_device_error()
        n = int(r["n_kept"][0])
        q.put((r["importance_local"].cpu().numpy(), r["ids"][0, :n].cpu().numpy(), r["out_tokens"][0, :n].cpu().numpy(),
               T[0].cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fused", "split"])
def test_dist_seq_path_single_rank(mode):
    """dist.seq_sharded_fused_specprefill (symmetric-memory rendezvous, peer
    buffers, sp_score_peer, sharded select) and the split path through an NCCL
    process group of one rank: the importance matches the oracle, the selection
    satisfies the parity rule, repeated calls give the same bits."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_dist_worker, args=(_free_port(), "C3", mode, q))
    p.start()
    try:
        imp, ids, out, tok = q.get(timeout=600)
    finally:
        p.join(timeout=120)
        if p.is_alive():
            p.kill()
    assert p.exitcode == 0
    w = gen.CONFIGS["C3"].with_(N=8192, R_valid=6)
    exact = _util.oracle_importance(w, 0)
    assert _util.rel_err(imp[0].astype(np.float64), exact) <= _util.REL_TOL
    o = ref.select(exact, w.keep, w.pool_k, w.chunk, 0)
    _util.check_selection(ids, ids, len(ids), o, w.chunk, w.N, 0)
    assert (out == tok[ids]).all()
