"""Multi-GPU partitions of the hot path: one process per GPU,
``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests) for the plumbing.

* Batch sharding -- requests are independent: rank p
  scores and selects its own requests with the single-GPU kernels, no
  collective on the data path.
* Head sharding -- the query heads (with their kv heads)
  split over the ranks: every lse is complete on its rank, the (l,h)-max is
  order-free, so the one exchange is an elementwise MAX all-reduce of
  acc2 [B][R_valid][N] (log2 domain), then importance = mean_r 2^acc2
  (sp_score_acc -> all_reduce(MAX) -> sp_acc_importance) and the selection.
* Sequence sharding, single pass (seq_sharded_fused_specprefill) -- the fused
  kernel exchanges the per-unit softmax statistics itself over peer memory
  (torch symmetric memory buffers, NVLink stores; sp_score_peer), so each rank
  reads its K shard once; then the sharded selection below.
* Sequence sharding, split (seq_sharded_specprefill) -- one request's prompt split along tokens.  The only real
  exchange is the softmax statistics (the lse of every (layer, head, row) needs
  all N keys):
    1. local statistics (m2, l) per row            (sp_score_stats)
    2. all-gather, merged in rank order -> lse2     (sp_stats_combine; identical on every rank)
    3. local importance with the global lse2        (sp_score_finish)
    4. the sharded selection below.
* Sequence-sharded selection (seq_sharded_select): the
  importance vector is never gathered.  Each rank pools its own chunks (the
  pooling windows reach (pool_k-1)/2 tokens into the neighbours: an all-gather
  of every rank's edge values), takes its local top-min(K_c, n_c/P) chunks as
  (score, chunk id) candidates, all-gathers them (8 B each) and every rank runs
  the same global top-K_c merge (sp_seq_edges -> all_gather -> sp_seq_candidates
  -> all_gather -> sp_seq_merge).  The ids/positions are bit-identical to
  sp_select_gather on the concatenated importance.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import api


def batch_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Requests [b0, b1) of rank `rank` (contiguous, sizes differ by at most 1)."""
    return rank * B // world, (rank + 1) * B // world


def token_range(N: int, world: int, rank: int, chunk: int = 1) -> tuple[int, int]:
    """Prompt tokens [i0, i1) of rank `rank` for sequence sharding; N must be a
    multiple of world (equal shards for the all-gathers)."""
    if N % world:
        raise ValueError(f"sequence sharding needs N ({N}) divisible by the number of ranks ({world})")
    n = N // world
    return rank * n, (rank + 1) * n


class CudaBackend:
    """The compute steps, all in libspecprefill.so kernels."""

    @staticmethod
    def score_stats(Q, K, R_valid, scale):
        return api.score_stats(Q, K, R_valid, scale)

    @staticmethod
    def stats_combine(parts):
        return api.stats_combine(parts)

    @staticmethod
    def score_finish(Q, K, lse2, R_valid, scale):
        return api.score_finish(Q, K, lse2, R_valid, scale)

    @staticmethod
    def score_acc(Q, K, R_valid, scale):
        return api.score_acc(Q, K, R_valid, scale)

    @staticmethod
    def acc_importance(acc2):
        return api.acc_importance(acc2)

    @staticmethod
    def select(imp, keep, pool_k, chunk, pos0, tokens):
        return api.select(imp, keep, pool_k, chunk, pos0, tokens=tokens)

    @staticmethod
    def seq_edges(imp_local, world, N, keep, pool_k, chunk):
        return api.seq_edges(imp_local, world, N, keep, pool_k, chunk)

    @staticmethod
    def seq_candidates(imp_local, edges_all, rank, world, N, keep, pool_k, chunk):
        return api.seq_candidates(imp_local, edges_all, rank, world, N, keep, pool_k, chunk)

    @staticmethod
    def seq_merge(cand_all, world, N, keep, pool_k, chunk, pos0, tokens):
        return api.seq_merge(cand_all, world, N, keep, pool_k, chunk, pos0, tokens=tokens)


def _all_gather(x: torch.Tensor, group) -> torch.Tensor:
    """[world][*x.shape] in rank order."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    if x.numel():
        dist.all_gather_into_tensor(out.view(-1), x.contiguous().view(-1), group=group)
    return out


def seq_sharded_select(imp_local, N_total: int, keep: float, pool_k: int, chunk: int, pos0: int = 0, tokens=None,
                       group=None, backend=None):
    """Selection over a sequence-sharded importance vector (imp_local [B][N/P]
    holds this rank's tokens, rank order = token order): edges all-gather,
    local candidates, candidate all-gather, global merge.  Returns (ids, pos,
    n_kept, out_tokens) for the whole prompt, identical on every rank; tokens
    [B][N_total] replicated (or None)."""
    be = backend or CudaBackend
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    edges = be.seq_edges(imp_local, world, N_total, keep, pool_k, chunk)              # [B][2w]
    edges_all = _all_gather(edges, group)                                               # [P][B][2w]
    cand = be.seq_candidates(imp_local, edges_all, rank, world, N_total, keep, pool_k, chunk)   # [B][M]
    cand_all = _all_gather(cand, group)                                                 # [P][B][M]
    r = be.seq_merge(cand_all, world, N_total, keep, pool_k, chunk, pos0, tokens)
    return r if tokens is not None else (*r, None)


def seq_sharded_specprefill(Q, K_local, tokens, N_total: int, keep: float, pool_k: int, chunk: int,
                            R_valid=None, scale=None, pos0: int = 0, group=None, backend=None) -> dict:
    """Sequence-sharded path for one request (B = 1).  Q [1][L][R][H][d] is
    replicated; K_local [1][L][Hkv][N_total/P][d] holds this rank's tokens
    (rank order = token order); tokens [1][N_total] int32 replicated.
    Returns importance_local [1][N_total/P] and ids, pos, n_kept, out_tokens
    for the whole prompt (identical on every rank)."""
    be = backend or CudaBackend
    world = dist.get_world_size(group)
    n_local = K_local.shape[3]
    if n_local * world != N_total or Q.shape[0] != 1:
        raise ValueError("K_local must hold N_total / world tokens of a single request")
    stats = be.score_stats(Q, K_local, R_valid, scale)                       # [rows][2]
    parts = torch.empty((world * stats.shape[0], 2), dtype=stats.dtype, device=stats.device)
    dist.all_gather_into_tensor(parts, stats.contiguous(), group=group)      # concatenated in rank order
    lse2 = be.stats_combine(parts.view(world, -1, 2))                        # [rows]
    imp_local = be.score_finish(Q, K_local, lse2, R_valid, scale)            # [1][n_local]
    ids, pos, n_kept, out = seq_sharded_select(imp_local, N_total, keep, pool_k, chunk, pos0, tokens, group, be)
    return dict(importance_local=imp_local, ids=ids, pos=pos, n_kept=n_kept, out_tokens=out,
                first_decode=N_total + pos0)


def head_range(Hkv: int, world: int, rank: int) -> tuple[int, int]:
    """kv heads [g0, g1) of rank `rank` for head sharding (query heads
    [g0*G, g1*G)); Hkv must be a multiple of world (equal head groups)."""
    if Hkv % world:
        raise ValueError(f"head sharding needs Hkv ({Hkv}) divisible by the number of ranks ({world})")
    n = Hkv // world
    return rank * n, (rank + 1) * n


def head_sharded_specprefill(Q_local, K_local, tokens, keep: float, pool_k: int, chunk: int, R_valid=None,
                             scale=None, pos0: int = 0, group=None, backend=None) -> dict:
    """Head-sharded path: Q_local [B][L][R][H/P][d] and K_local [B][L][Hkv/P][N][d]
    hold this rank's heads (head_range); tokens [B][N] replicated.  The scale
    must be given explicitly (it depends on d only, but keep it the caller's).
    Returns importance [B][N], ids, pos, n_kept, out_tokens (replicated)."""
    be = backend or CudaBackend
    acc2 = be.score_acc(Q_local, K_local, R_valid, scale)                      # [B][Rv][N]
    dist.all_reduce(acc2, op=dist.ReduceOp.MAX, group=group)                  # order-free: exact
    imp = be.acc_importance(acc2.contiguous())
    ids, pos, n_kept, out = be.select(imp, keep, pool_k, chunk, pos0, tokens)
    N = imp.shape[1]
    return dict(importance=imp, ids=ids, pos=pos, n_kept=n_kept, out_tokens=out, first_decode=N + pos0)


_PEER_CACHE: dict = {}


def _peer_buffers(Q, K_local, R_valid, group):
    """This rank's partial buffer in torch symmetric memory, every rank's
    address of it, and the launch workspace that goes with it (cached per
    geometry, never evicted).  The workspace's launch epoch picks the half of
    the partial buffers a launch writes, so both are created zeroed together
    and live together: a fresh epoch never meets stale partials."""
    import torch.distributed._symmetric_memory as symm_mem
    world = dist.get_world_size(group)
    key = (tuple(K_local.shape), tuple(Q.shape), R_valid, world, id(group), K_local.device.index)
    if key not in _PEER_CACHE:
        nbytes = api.score_peer_buffer_bytes(Q, K_local, world, 0, R_valid)
        buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=K_local.device)
        buf.zero_()
        pg = group if group is not None else dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, pg.group_name)
        ws = torch.zeros(max(256, api.score_peer_workspace_bytes(Q, K_local, world, 0, R_valid)), dtype=torch.uint8,
                         device=K_local.device)
        torch.cuda.synchronize()
        dist.barrier(group)
        _PEER_CACHE[key] = (buf, hdl, [int(x) for x in hdl.buffer_ptrs], ws)
    _, _, ptrs, ws = _PEER_CACHE[key]
    return ptrs, ws


def seq_sharded_fused_specprefill(Q, K_local, tokens, N_total: int, keep: float, pool_k: int, chunk: int,
                                  R_valid=None, scale=None, pos0: int = 0, group=None, check: bool = True) -> dict:
    """Sequence-sharded single pass for one request (B = 1): the statistics
    exchange runs inside the fused kernel over peer memory (one K read per
    rank); the edge all-gather of the sharded selection that follows also
    separates consecutive calls (sp_score_peer's barrier requirement: no rank
    starts the next launch before every rank's kernel finished).  check: read
    the device error flag at the end (synchronises the stream) so a peer that
    never arrived (SP_ETIMEOUT: its words merged as empty) raises instead of
    returning a silently wrong selection."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_local = K_local.shape[3]
    if n_local * world != N_total or Q.shape[0] != 1:
        raise ValueError("K_local must hold N_total / world tokens of a single request")
    ptrs, ws = _peer_buffers(Q, K_local, R_valid, group)
    imp_local = api.score_peer(Q, K_local, rank, world, ptrs, 0, R_valid, scale, ws=ws)
    ids, pos, n_kept, out = seq_sharded_select(imp_local, N_total, keep, pool_k, chunk, pos0, tokens, group)
    if check:
        api.check_device_error()
    return dict(importance_local=imp_local, ids=ids, pos=pos, n_kept=n_kept, out_tokens=out,
                first_decode=N_total + pos0)


def batch_sharded_specprefill(Q, K, tokens, keep, pool_k, chunk, R_valid=None, scale=None, pos0=0) -> dict:
    """Batch sharding: the caller passes this rank's requests; no collective."""
    return api.specprefill(Q, K, tokens, keep, pool_k, chunk, R_valid, scale, pos0)
