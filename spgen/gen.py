"""Counter-based synthetic inputs (numpy side).  No method arithmetic lives here.

Every element is a pure function of (seed, stream, global index), computed with
64-bit integer hashing (splitmix64 finaliser) and small-integer arithmetic, so
``spgen/gen.cu`` reproduces it bit for bit and any slice (one (b, l, kv-head)
unit, one token range of a sequence shard) can be regenerated on its own.

Values.  Every K / Q element is ``v = k_int / 64`` with ``|k_int| <= 255``;
such values are exactly representable in bf16 (8 significant bits), so there
is no rounding anywhere and the bf16 bit pattern is simply the top half of the
float32 bit pattern of ``v``.

Structure:
* background keys ~ Irwin-Hall(4) of 7-bit uniforms, sigma ~= 1.15;
* per (b, l, kv-head) a +-1 "direction" u[t]; queries of that group are
  ``amp * u + noise/2`` with amp 1.0 for one head in four (retrieval-like heads)
  and 0.25 otherwise, so look-ahead rows are correlated;
* attention sink: tokens 0..3 get ``+1.5 u`` (sink phenomenon);
* proximity bias: a trailing ramp ``+0.5 (i/N)^2 u``;
* needles: 1-4 spans of 16-64 tokens at seeded positions, ``+1.0 u`` on a
  seeded 10% of (l, kv-head) units (RULER NIAH-like);
* outlier channels: ~d/64 channels per unit with a near-constant +-3.1 value
  (Llama K-cache outlier channels; softmax-shift invariant).

Value modes (``Workload.values``):
* ``"dyadic"`` (default) -- the k/64 grid above: every bf16 product and every
  fp32 dot-product partial sum is exact, so the selection's tie-break can be
  tested bit-exactly;
* ``"randn"`` -- full-mantissa bf16: each value is an integer in units of 2^-15
  (noise = sum of four 16-bit uniforms, sigma ~= 1.15; the same structure
  amplitudes x 512), converted exactly to float32 and rounded to bf16
  (round-to-nearest-even on the bit pattern), so products carry all 8
  significand bits and fp32 accumulation rounds as it does on real caches.
  Outlier channels are 4x larger (+-12.5) and one query head in sixteen is an
  "outlier head" (amplitude 2.5: logits of ~40 on the sink tokens).

Planted tiers (``Workload.planted``): a fixture in which every keep rate of the
C4 sweep (i/10, i = 1..9) has a clear K_c boundary.  Chunks are ranked by a
seeded permutation (chunk 0, the sink chunk, first) and cut into ten tiers at
K_c(i/10); the interior tokens [w, chunk - w) of a tier-t chunk (w =
(pool_k - 1) / 2, so pooling never carries a boost across a chunk edge) get
``+(PLANT_BASE + PLANT_STEP * t) u``.  Needles and the proximity ramp are off.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# ---------------------------------------------------------------- hashing
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_M64 = (1 << 64) - 1

# stream ids (must match gen.cu)
S_KNOISE, S_USIGN, S_QNOISE, S_HEADAMP, S_OUTLIER, S_NEEDLE_LG, S_TOKENS, S_SPANS = 1, 2, 3, 4, 5, 6, 7, 8

# structure amplitudes in 1/64 units (must match gen.cu)
SINK_TOKENS = 4
SINK_AMP = 96          # +1.5
RAMP_AMP = 32          # up to ~+0.5
NEEDLE_AMP = 64        # +1.0
OUTLIER_AMP = 200      # +-3.125
QA_STRONG = 64         # 1.0
QA_WEAK = 16           # 0.25
VOCAB = 128256         # Llama-3 vocabulary size (token ids for the gather)
MIN_N_FOR_NEEDLES = 256
# "randn" mode (units of 2^-15; the dyadic amplitudes x 512)
RN_UNIT = 512
RN_OUTLIER = 4 * OUTLIER_AMP * RN_UNIT     # +-12.5
RN_QA_OUTLIER = 160 * RN_UNIT              # 2.5: "outlier" query heads (one in sixteen)
# planted tiers (1/64 units; x 512 in randn mode)
PLANT_TIERS = 10
PLANT_BASE = 40
PLANT_STEP = 4
S_PLANT = 9


def _mix_int(x: int) -> int:
    """splitmix64 finaliser on a Python int (mod 2^64)."""
    x &= _M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    x ^= x >> 31
    return x


def stream_key(seed: int, stream: int) -> int:
    return _mix_int(((seed & _M64) * 0x9E3779B97F4A7C15 + stream) & _M64)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * _C1
    x = x ^ (x >> np.uint64(27))
    x = x * _C2
    x = x ^ (x >> np.uint64(31))
    return x


def h64(key: int, idx) -> np.ndarray:
    """hash(key, idx) = mix(idx * GOLD + key), all mod 2^64."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(idx * _GOLD + np.uint64(key))


def _noise4(h: np.ndarray) -> np.ndarray:
    """Sum of four 7-bit fields minus 254: integer in [-254, 254]."""
    m = np.uint64(127)
    s = (h & m) + ((h >> np.uint64(8)) & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(24)) & m)
    return s.astype(np.int64) - 254


def _noise16(h: np.ndarray) -> np.ndarray:
    """Sum of four 16-bit fields minus 2*65535: integer in [-131070, 131070]."""
    m = np.uint64(0xFFFF)
    s = (h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + ((h >> np.uint64(48)) & m)
    return s.astype(np.int64) - 131070


def _rn_to_bf16_bits(vint: np.ndarray) -> np.ndarray:
    """v * 2^-15 -> bf16, round to nearest even (|v| < 2^24: the float32 value is exact)."""
    f = vint.astype(np.float32) * np.float32(2.0 ** -15)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return b.astype(np.uint16)


def _to_bf16_bits(vint: np.ndarray) -> np.ndarray:
    """k_int/64 -> bf16 bit pattern (exact: |k_int| <= 255)."""
    f = vint.astype(np.float32) / np.float32(64.0)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


# ---------------------------------------------------------------- workloads
@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (or a test variant of it)."""
    name: str
    B: int
    L: int
    H: int
    Hkv: int
    d: int
    N: int
    R: int
    keep: float
    pool_k: int
    chunk: int
    R_valid: int | None = None
    seed: int = 0
    pos0: int = 0
    values: str = "dyadic"        # "dyadic" (k/64, exact products) | "randn" (full-mantissa bf16)
    planted: bool = False         # planted-tier fixture (clear K_c boundaries at keep i/10)

    @property
    def G(self) -> int:
        return self.H // self.Hkv

    @property
    def Rv(self) -> int:
        return self.R if self.R_valid is None else self.R_valid

    @property
    def scale(self) -> float:
        """Softmax scale 1/sqrt(d) (reading Z3), rounded to float32 because the
        C ABI carries it as a float; both sides use this exact value."""
        return float(np.float32(1.0 / math.sqrt(self.d)))

    @property
    def n_chunks(self) -> int:
        return -(-self.N // self.chunk)

    @property
    def k_bytes(self) -> int:
        return self.B * self.L * self.Hkv * self.N * self.d * 2

    @property
    def q_bytes(self) -> int:
        return self.B * self.L * self.R * self.H * self.d * 2

    def with_(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; chunk 32 / pool 5 for the 8B configs and
# R=8 for C2-C4 are DESIGN.md readings Z7 / Z1 (the paper states neither).
CONFIGS = {
    "C0": Workload("tiny", B=1, L=2, H=4, Hkv=2, d=16, N=64, R=2, keep=0.5, pool_k=3, chunk=4),
    "C1": Workload("8b-4k", B=1, L=32, H=32, Hkv=8, d=128, N=4096, R=8, keep=0.1, pool_k=5, chunk=32),
    "C2": Workload("8b-64x1k", B=64, L=32, H=32, Hkv=8, d=128, N=1024, R=8, keep=0.3, pool_k=5, chunk=32),
    "C3": Workload("8b-32k", B=1, L=32, H=32, Hkv=8, d=128, N=32768, R=8, keep=0.1, pool_k=5, chunk=32),
    "C4": Workload("8b-128k", B=1, L=32, H=32, Hkv=8, d=128, N=131072, R=8, keep=0.1, pool_k=5, chunk=32),
}


# ---------------------------------------------------------------- structure tables
def needle_spans(w: Workload, b: int) -> list[tuple[int, int]]:
    """Seeded needle spans [start, end) of request b (global token indices)."""
    if w.N < MIN_N_FOR_NEEDLES:
        return []
    key = stream_key(w.seed, S_SPANS)
    hs = [int(x) for x in h64(key, np.arange(b * 16, b * 16 + 16, dtype=np.uint64))]
    count = 1 + hs[0] % 4
    spans = []
    for j in range(count):
        length = 16 + hs[1 + 2 * j] % 49
        start = hs[2 + 2 * j] % (w.N - length)
        spans.append((start, start + length))
    return sorted(spans)


def _usign(w: Workload, b: int, l: int, g, t) -> np.ndarray:
    key = stream_key(w.seed, S_USIGN)
    idx = ((np.uint64(b) * np.uint64(w.L) + np.uint64(l)) * np.uint64(w.Hkv) + np.asarray(g, np.uint64)) \
        * np.uint64(w.d) + np.asarray(t, np.uint64)
    return 1 - 2 * (h64(key, idx) & np.uint64(1)).astype(np.int64)


def planted_tiers(w: Workload, b: int) -> np.ndarray:
    """Tier (0..9) of every chunk of request b in the planted fixture: chunks
    ranked by a seeded permutation (chunk 0 first), ten tiers cut at positions
    ceil(j * n_c / 10), j = 1..9 (the top tier rounds up); tier 9 is the top."""
    n_c = w.n_chunks
    order = np.argsort(h64(stream_key(w.seed, S_PLANT), np.uint64(b) * np.uint64(n_c)
                           + np.arange(n_c, dtype=np.uint64)), kind="stable")
    order = np.concatenate([[0], order[order != 0]])
    cuts = np.array([(j * n_c + PLANT_TIERS - 1) // PLANT_TIERS for j in range(1, PLANT_TIERS)])
    tier_of_rank = (PLANT_TIERS - 1) - np.searchsorted(cuts, np.arange(n_c), side="right")
    tiers = np.empty(n_c, dtype=np.int64)
    tiers[order] = tier_of_rank
    return tiers


def _unit_scale(w: Workload) -> int:
    return RN_UNIT if w.values == "randn" else 1


# ---------------------------------------------------------------- generators
def gen_K_int(w: Workload, b: int, l: int, g: int, i0: int = 0, i1: int | None = None) -> np.ndarray:
    """Integer K values of unit (b, l, g), tokens [i0, i1): [n, d] int64, in
    units of 1/64 ("dyadic") or 2^-15 ("randn")."""
    i1 = w.N if i1 is None else i1
    d = w.d
    rn = w.values == "randn"
    us = _unit_scale(w)
    i = np.arange(i0, i1, dtype=np.uint64)[:, None]
    t = np.arange(d, dtype=np.uint64)[None, :]
    unit = (b * w.L + l) * w.Hkv + g
    with np.errstate(over="ignore"):
        idx = ((np.uint64(unit) * np.uint64(w.N) + i) * np.uint64(d)) + t
    hn = h64(stream_key(w.seed, S_KNOISE), idx)
    n = _noise16(hn) if rn else _noise4(hn)
    u = _usign(w, b, l, g, np.arange(d, dtype=np.uint64))[None, :]
    ii = np.arange(i0, i1, dtype=np.int64)[:, None]
    k = n.copy()
    k += np.where(ii < SINK_TOKENS, SINK_AMP * us, 0) * u
    if w.planted:
        tiers = planted_tiers(w, b)
        c = ii // w.chunk
        j = ii - c * w.chunk
        hw = (w.pool_k - 1) // 2
        tt = tiers[c]
        boost = np.where((tt > 0) & (j >= hw) & (j < w.chunk - hw), (PLANT_BASE + PLANT_STEP * tt) * us, 0)
        k += boost * u
    else:
        r = (ii * 64) // w.N
        k += (r * r * 4 if rn else (RAMP_AMP * r * r) >> 12) * u
        nlg = int(h64(stream_key(w.seed, S_NEEDLE_LG), np.uint64(unit))) % 10 == 0
        if nlg:
            inside = np.zeros_like(ii, dtype=bool)
            for (s, e) in needle_spans(w, b):
                inside |= (ii >= s) & (ii < e)
            k += np.where(inside, NEEDLE_AMP * us, 0) * u
    ho = h64(stream_key(w.seed, S_OUTLIER), np.uint64(unit) * np.uint64(d) + np.arange(d, dtype=np.uint64))
    is_out = (ho % np.uint64(64)) == 0
    osign = 1 - 2 * ((ho >> np.uint64(32)) & np.uint64(1)).astype(np.int64)
    k = np.where(is_out[None, :], osign[None, :] * (RN_OUTLIER if rn else OUTLIER_AMP) + (n >> 3), k)
    return k if rn else np.clip(k, -255, 255)


def _bits(w: Workload, vint: np.ndarray) -> np.ndarray:
    return _rn_to_bf16_bits(vint) if w.values == "randn" else _to_bf16_bits(vint)


def gen_K(w: Workload, b: int, l: int, g: int, i0: int = 0, i1: int | None = None) -> np.ndarray:
    """bf16 bit patterns (uint16) of K[b][l][g][i0:i1][:]."""
    return _bits(w, gen_K_int(w, b, l, g, i0, i1))


def gen_Q_int(w: Workload, b: int, l: int) -> np.ndarray:
    """Integer Q values of request b, layer l: [R, H, d] int64 (units as gen_K_int)."""
    R, H, d = w.R, w.H, w.d
    rn = w.values == "randn"
    us = _unit_scale(w)
    r = np.arange(R, dtype=np.uint64)[:, None, None]
    h = np.arange(H, dtype=np.uint64)[None, :, None]
    t = np.arange(d, dtype=np.uint64)[None, None, :]
    with np.errstate(over="ignore"):
        idx = (((np.uint64(b) * np.uint64(w.L) + np.uint64(l)) * np.uint64(R) + r) * np.uint64(H) + h) \
            * np.uint64(d) + t
    hq = h64(stream_key(w.seed, S_QNOISE), idx)
    nq = (_noise16(hq) if rn else _noise4(hq)) >> 1
    g = np.arange(H, dtype=np.uint64) // np.uint64(w.G)
    u = _usign(w, b, l, g[:, None], np.arange(d, dtype=np.uint64)[None, :])      # [H, d]
    ha = h64(stream_key(w.seed, S_HEADAMP), np.uint64(b * w.L + l) * np.uint64(H) + np.arange(H, dtype=np.uint64))
    amp = np.where((ha % np.uint64(4)) == 0, QA_STRONG * us, QA_WEAK * us).astype(np.int64)  # [H]
    if rn:
        amp = np.where((ha % np.uint64(16)) == 1, RN_QA_OUTLIER, amp)
    q = amp[None, :, None] * u[None, :, :] + nq
    return q if rn else np.clip(q, -255, 255)


def gen_Q(w: Workload, b: int, l: int) -> np.ndarray:
    """bf16 bit patterns (uint16) of Q[b][l][:R][:H][:d]."""
    return _bits(w, gen_Q_int(w, b, l))


def gen_tokens(w: Workload, b: int, i0: int = 0, i1: int | None = None) -> np.ndarray:
    i1 = w.N if i1 is None else i1
    idx = np.uint64(b) * np.uint64(w.N) + np.arange(i0, i1, dtype=np.uint64)
    return (h64(stream_key(w.seed, S_TOKENS), idx) % np.uint64(VOCAB)).astype(np.int32)


def gen_request(w: Workload, b: int):
    """Whole request b as bf16 bits: Q [L][R][H][d], K [L][Hkv][N][d]; tokens [N]."""
    Q = np.stack([gen_Q(w, b, l) for l in range(w.L)])
    K = np.stack([np.stack([gen_K(w, b, l, g) for g in range(w.Hkv)]) for l in range(w.L)])
    return Q, K, gen_tokens(w, b)


def gen_batch(w: Workload):
    """Whole batch as bf16 bits: Q [B][L][R][H][d], K [B][L][Hkv][N][d], tokens [B][N]."""
    reqs = [gen_request(w, b) for b in range(w.B)]
    return (np.stack([r[0] for r in reqs]), np.stack([r[1] for r in reqs]), np.stack([r[2] for r in reqs]))
