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

    # sequence-sharded selection, restated with the oracle's O5-O9 on one shard
    @staticmethod
    def seq_edges(imp_local, world, N, keep, pool_k, chunk):
        w = (pool_k - 1) // 2
        n = imp_local.shape[1]
        return torch.cat([imp_local[:, :w], imp_local[:, n - w:]], dim=1)

    @staticmethod
    def seq_candidates(imp_local, edges_all, rank, world, N, keep, pool_k, chunk):
        """Local pooled chunk scores (windows completed with the neighbours'
        edges) and the local top-min(K_c, n_c/P) chunks as (global id, score)."""
        w = (pool_k - 1) // 2
        n = imp_local.shape[1]
        K_c = ref.kept_chunk_count(-(-N // chunk), keep)
        M = min(K_c, n // chunk)
        out = []
        for b in range(imp_local.shape[0]):
            parts = [imp_local[b].numpy()]
            if rank > 0:
                parts.insert(0, edges_all[rank - 1, b, w:].numpy())
            if rank + 1 < world:
                parts.append(edges_all[rank + 1, b, :w].numpy())
            ext = np.concatenate(parts)                                 # the array's ends are true sequence ends
            off = w if rank > 0 else 0
            cs = ref.chunk_scores(ref.smooth_scores(ext, pool_k)[off:off + n], chunk)
            kept = ref.select_chunks(cs, M)
            out.append(np.stack([kept + rank * (n // chunk), cs[kept]], axis=1))
        return torch.tensor(np.stack(out))                              # [B][M][2]

    @staticmethod
    def seq_merge(cand_all, world, N, keep, pool_k, chunk, pos0, tokens):
        n_c = -(-N // chunk)
        K_c = ref.kept_chunk_count(n_c, keep)
        B = cand_all.shape[1]
        ids_all = torch.zeros((B, N), dtype=torch.int64)
        nk = torch.zeros(B, dtype=torch.int64)
        outs = torch.zeros((B, N), dtype=torch.int64)
        for b in range(B):
            cs = np.full(n_c, -np.inf)
            c = cand_all[:, b].reshape(-1, 2).numpy()
            cs[c[:, 0].astype(np.int64)] = c[:, 1]
            kept = ref.select_chunks(cs, K_c)
            ids, _, _ = ref.restore_position_ids(kept, chunk, N, pos0)
            ids_all[b, :len(ids)] = torch.tensor(ids)
            nk[b] = len(ids)
            if tokens is not None:
                outs[b, :len(ids)] = torch.tensor(ref.gather(tokens[b].numpy(), ids))
        return ids_all, ids_all + pos0, nk, outs


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
        imp = r["importance_local"] if mode == "seq" else r["importance"]
        outq.put((rank, imp.numpy(), r["ids"].numpy(), int(r["n_kept"][0]), r["out_tokens"].numpy()))
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
        i0, i1 = (rank * w.N // world, (rank + 1) * w.N // world) if mode == "seq" else (0, w.N)
        np.testing.assert_allclose(imp[0], o["imp"][i0:i1], rtol=1e-12)
        assert n == o["n_kept"]
        np.testing.assert_array_equal(ids[0][:n], o["ids"])
        np.testing.assert_array_equal(out[0][:n], o["out_tokens"])


def _select_worker(rank, world, port, N, cases, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_02789_b200 import dist as spd
        res = []
        for (imp, keep, pool_k, chunk, pos0) in cases:
            i0, i1 = spd.token_range(N, world, rank)
            tok = torch.tensor(np.arange(N, dtype=np.int64) * 7 + 3)[None]
            ids, pos, nk, out = spd.seq_sharded_select(torch.tensor(imp[None, i0:i1]), N, keep, pool_k, chunk, pos0,
                                                       tok, backend=OracleBackend)
            n = int(nk[0])
            res.append((ids[0, :n].numpy(), pos[0, :n].numpy(), out[0, :n].numpy()))
        outq.put((rank, res))
    finally:
        dist.destroy_process_group()


def _seq_select_cases(N, world):
    """Importance vectors whose chunk scores tie across ranks (dyadic values:
    float64 sums are exact), over keep rates below and above 1/P."""
    rng = np.random.default_rng(5)
    cases = []
    for chunk, pool_k in [(8, 5), (4, 1), (16, 9), (1, 3)]:
        n_c = N // chunk
        per = rng.integers(1, 6, size=n_c // world)                      # chunk level pattern, repeated per rank
        lev = np.tile(per, world).astype(np.float64)
        imp = np.repeat(lev, chunk) / 8.0                                 # constant chunks: ties across ranks
        for keep in (0.1, 1.0 / world, 0.5, 0.9):
            cases.append((imp, keep, pool_k, chunk, 11))
        noisy = imp + rng.integers(0, 3, size=N) / 64.0                   # near-ties, still dyadic
        cases.append((noisy, 0.3, pool_k, chunk, 0))
    return cases


@pytest.mark.parametrize("world", [2, 4])
def test_seq_sharded_select_gloo(world):
    """Row e: edges all-gather -> local top-min(K_c,
    n_c/P) candidates -> candidate all-gather -> global merge gives exactly the
    oracle's whole-prompt selection on every rank, including chunk-score ties
    across ranks (lowest index wins) and keep rates >= 1/P."""
    N = 256
    cases = _seq_select_cases(N, world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_select_worker, args=(r, world, port, N, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=240) for _ in range(world))    # drain before join (large queue items)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert [p.exitcode for p in procs] == [0] * world
    for k, (imp, keep, pool_k, chunk, pos0) in enumerate(cases):
        o = ref.select(imp, keep, pool_k, chunk, pos0)
        for rank in range(world):
            ids, pos, out = res[rank][k]
            np.testing.assert_array_equal(ids, o["ids"], err_msg=f"case {k} rank {rank}")
            np.testing.assert_array_equal(pos, o["pos"])
            np.testing.assert_array_equal(out, o["ids"] * 7 + 3)


def test_ranges():
    from paper_2502_02789_b200 import dist as spd
    assert [spd.batch_range(10, 4, r) for r in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    assert [spd.token_range(32768, 8, r) for r in (0, 7)] == [(0, 4096), (28672, 32768)]
    with pytest.raises(ValueError):
        spd.token_range(1000, 3, 0)
    assert [spd.head_range(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        spd.head_range(8, 3, 0)
