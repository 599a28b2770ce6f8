"""Multi-process (gloo, world_size 2) tests of the sequence- and head-sharded
choreographies on CPU.  The CUDA kernels cannot run here, so the compute steps are injected
as a float64 backend restating the oracle in split form; the collectives,
shard boundaries, rank-order merges and the final selection are the product's
(paper_2502_02789_b200.dist)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref
from spgen import gen

LOG2E = 1.0 / math.log(2.0)


class OracleBackend:
    """float64 restatement of O1-O4 split at the statistics exchange (log2 domain)."""

    @staticmethod
    def _logits2(Q, K, scale):
        L, R, H, d = Q.shape[1:]
        Hkv = K.shape[2]
        G = H // Hkv
        x = np.empty((L, H, R, K.shape[3]))
        for l in range(L):
            for h in range(H):
                x[l, h] = scale * LOG2E * (Q[0, l, :, h, :].numpy() @ K[0, l, h // G].numpy().T)
        return x

    @classmethod
    def score_stats(cls, Q, K, R_valid, scale):
        x = cls._logits2(Q[:, :, :R_valid], K, scale)                  # [L][H][Rv][n]
        m = x.max(axis=3)
        s = np.exp2(x - m[..., None]).sum(axis=3)
        return torch.tensor(np.stack([m.reshape(-1), s.reshape(-1)], axis=1))

    @staticmethod
    def stats_combine(parts):
        p = parts.numpy()
        M = p[:, :, 0].max(axis=0)
        S = np.zeros_like(M)
        for r in range(p.shape[0]):                                     # rank order
            S += p[r, :, 1] * np.exp2(p[r, :, 0] - M)
        return torch.tensor(M + np.log2(S))

    @classmethod
    def score_finish(cls, Q, K, lse2, R_valid, scale):
        x = cls._logits2(Q[:, :, :R_valid], K, scale)
        L, H, Rv, n = x.shape
        t = x - lse2.numpy().reshape(L, H, Rv)[..., None]
        acc = t.max(axis=1).max(axis=0)                                 # [Rv][n]
        return torch.tensor(np.exp2(acc).mean(axis=0))[None]

    @classmethod
    def score_acc(cls, Q, K, R_valid, scale):
        x = cls._logits2(Q[:, :, :R_valid], K, scale)                  # [L][H/P][Rv][N], local heads
        m = x.max(axis=3, keepdims=True)
        lse2 = m + np.log2(np.exp2(x - m).sum(axis=3, keepdims=True))  # complete: all tokens are local
        return torch.tensor((x - lse2).max(axis=1).max(axis=0))[None]  # [1][Rv][N]

    @staticmethod
    def acc_importance(acc2):
        return torch.tensor(np.exp2(acc2.numpy()).mean(axis=1))        # [1][N]

    @staticmethod
    def select(imp, keep, pool_k, chunk, pos0, tokens):
        r = ref.select(imp[0].numpy(), keep, pool_k, chunk, pos0)
        ids = torch.tensor(r["ids"])[None]
        return ids, ids + pos0, torch.tensor([r["n_kept"]]), torch.tensor(ref.gather(tokens[0].numpy(), r["ids"]))[None]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, w, outq, mode="seq"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_02789_b200 import dist as spd
        Qb, Kb, tok = gen.gen_batch(w)
        if mode == "seq":
            Q = torch.tensor(ref.bf16_to_f64(Qb))
            i0, i1 = spd.token_range(w.N, world, rank)
            K = torch.tensor(ref.bf16_to_f64(Kb[:, :, :, i0:i1]))
            r = spd.seq_sharded_specprefill(Q, K, torch.tensor(tok), w.N, w.keep, w.pool_k, w.chunk, w.Rv, w.scale,
                                            w.pos0, backend=OracleBackend)
        else:
            g0, g1 = spd.head_range(w.Hkv, world, rank)
            Q = torch.tensor(ref.bf16_to_f64(Qb[:, :, :, g0 * w.G:g1 * w.G]))
            K = torch.tensor(ref.bf16_to_f64(Kb[:, :, g0:g1]))
            r = spd.head_sharded_specprefill(Q, K, torch.tensor(tok), w.keep, w.pool_k, w.chunk, w.Rv, w.scale,
                                             w.pos0, backend=OracleBackend)
        outq.put((rank, r["importance"].numpy(), r["ids"].numpy(), int(r["n_kept"][0]), r["out_tokens"].numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["seq", "head"])
@pytest.mark.parametrize("world", [2])
def test_sharded_choreography_gloo(world, mode):
    """Sequence sharding (statistics all-gather) and head sharding (MAX
    all-reduce of the log-domain maxima, row f1) give the oracle's result on
    every rank."""
    w = gen.CONFIGS["C0"].with_(N=256, L=3, R=3, R_valid=2, chunk=8, pos0=5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0] * world, codes
    res = [q.get(timeout=10) for _ in range(world)]
    Qb, Kb, tok = gen.gen_batch(w)
    o = ref.specprefill(Qb[0], Kb[0], tok[0], w.scale, w.keep, w.pool_k, w.chunk, w.Rv, w.pos0)
    for rank, imp, ids, n, out in res:
        np.testing.assert_allclose(imp[0], o["imp"], rtol=1e-12)
        assert n == o["n_kept"]
        np.testing.assert_array_equal(ids[0][:n], o["ids"])
        np.testing.assert_array_equal(out[0][:n], o["out_tokens"])


def test_ranges():
    from paper_2502_02789_b200 import dist as spd
    assert [spd.batch_range(10, 4, r) for r in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    assert [spd.token_range(32768, 8, r) for r in (0, 7)] == [(0, 4096), (28672, 32768)]
    with pytest.raises(ValueError):
        spd.token_range(1000, 3, 0)
    assert [spd.head_range(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        spd.head_range(8, 3, 0)
