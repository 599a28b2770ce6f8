"""Paged K-cache layout for SURVEY 8(f) row f3 -- test/bench infrastructure.

Layout only (no method arithmetic): contiguous K [B][L][Hkv][N][d] scattered
into a vLLM-style cache [L][num_blocks][block_size][Hkv][d] through a seeded,
shuffled block table (plus a few spare, NaN-filled blocks no request owns).
"""
from __future__ import annotations

import torch


def to_paged(K: torch.Tensor, bs: int, seed: int = 0, spare: int = 3, layout: str = "nhd"):
    """Returns (cache [L][nblk][bs][Hkv][d], block_table int32 [B][ceil(N/bs)]).

    layout "nhd": blocks stored [bs][Hkv][d] (vLLM's flash-attention layout:
    the kv heads of a token interleaved); "hnd": stored [Hkv][bs][d] (FlashInfer's
    HND layout: a head's block rows contiguous), returned as the same
    [L][nblk][bs][Hkv][d] view with the corresponding strides."""
    B, L, Hkv, N, d = K.shape
    mb = -(-N // bs)
    nblk = B * mb + spare
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(nblk, generator=g)[:B * mb].view(B, mb)
    fill = 0x7F if K.dtype == torch.uint8 else float("nan")          # (e4m3 codes: 0x7F is NaN)
    if layout == "hnd":
        store = torch.full((L, nblk, Hkv, bs, d), fill, dtype=K.dtype, device=K.device)
        cache = store.permute(0, 1, 3, 2, 4)
    else:
        cache = torch.full((L, nblk, bs, Hkv, d), fill, dtype=K.dtype, device=K.device)
    for b in range(B):
        Kp = torch.nn.functional.pad(K[b], (0, 0, 0, mb * bs - N))                 # [L][Hkv][mb*bs][d]
        Kp = Kp.view(L, Hkv, mb, bs, d).permute(0, 2, 3, 1, 4)                     # [L][mb][bs][Hkv][d]
        cache[:, perm[b].to(K.device)] = Kp
    return cache, perm.to(torch.int32).to(K.device)
