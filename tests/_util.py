"""Shared test helpers: oracle runs on generated inputs and the parity rule."""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

from oracle import ref
from spgen import gen

REL_TOL = 1e-3          # importance / chunk-score tolerance (BASELINE.json north_star)
_POOL = cf.ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)))

# Parity report ("report the fraction of (config, seed, keep) cases
# in each regime"): every full-size case appends a record; tests/conftest.py
# prints the table at the end of the session and writes gpurun_out/parity_regimes.json.
RECORDS: list[dict] = []


def record(w: gen.Workload, keep: float, b: int, regime: str, margin: float, rel_err: float, where: str):
    RECORDS.append(dict(where=where, config=w.name, N=w.N, B=w.B, seed=w.seed, values=w.values,
                        planted=w.planted, request=b, keep=keep, regime=regime,
                        margin=None if margin == float("inf") else float(margin), max_rel_err=float(rel_err)))


def k_layer_f64(w: gen.Workload, b: int, l: int, i0: int = 0, i1: int | None = None) -> np.ndarray:
    """K[b][l] as float64 [Hkv][n][d], kv heads generated in parallel."""
    parts = list(_POOL.map(lambda g: ref.bf16_to_f64(gen.gen_K(w, b, l, g, i0, i1)), range(w.Hkv)))
    return np.stack(parts)


def oracle_importance(w: gen.Workload, b: int) -> np.ndarray:
    Q = ref.bf16_to_f64(np.stack([gen.gen_Q(w, b, l) for l in range(w.L)]))
    return ref.token_importance(Q, lambda l: k_layer_f64(w, b, l), w.scale, w.Rv)


def oracle_request(w: gen.Workload, b: int, keep: float | None = None) -> dict:
    imp = oracle_importance(w, b)
    r = ref.select(imp, w.keep if keep is None else keep, w.pool_k, w.chunk, w.pos0)
    r["imp"] = imp
    return r


def rel_err(gpu: np.ndarray, exact: np.ndarray) -> float:
    return float(np.max(np.abs(gpu - exact) / np.maximum(np.abs(exact), 1e-30)))


def check_selection(ids: np.ndarray, pos: np.ndarray, n_kept: int, o: dict, chunk: int, N: int, pos0: int) -> str:
    """DESIGN.md parity rule for one request.  Returns the regime ("exact" when
    the K_c-th margin exceeds the tolerance, else "near-tie")."""
    ids = np.asarray(ids[:n_kept], dtype=np.int64)
    pos = np.asarray(pos[:n_kept], dtype=np.int64)
    assert (np.diff(ids) > 0).all(), "ids must be strictly ascending"
    np.testing.assert_array_equal(pos, ids + pos0)
    m = ref.margin(o["cs"], o["K_c"])
    if m > REL_TOL:
        assert n_kept == o["n_kept"], (n_kept, o["n_kept"])
        np.testing.assert_array_equal(ids, o["ids"])
        return "exact"
    # near-tie: a valid top-K_c set under the oracle scores within tolerance
    kept_c = np.unique(ids // chunk)
    assert len(kept_c) == o["K_c"]
    sizes = np.minimum((kept_c + 1) * chunk, N) - kept_c * chunk
    assert n_kept == int(sizes.sum())
    # whole chunks, in order: ids are exactly the concatenated token ranges of the kept chunks
    starts = np.repeat(kept_c * chunk, sizes)
    offs = np.arange(n_kept) - np.repeat(np.cumsum(sizes) - sizes, sizes)
    np.testing.assert_array_equal(ids, starts + offs)
    cs = o["cs"]
    dropped = np.setdiff1d(np.arange(len(cs)), kept_c)
    if len(dropped):
        assert cs[kept_c].min() >= cs[dropped].max() * (1 - REL_TOL)
    return "near-tie"
