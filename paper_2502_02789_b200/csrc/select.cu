// Selection: 1-D average pool -> chunk means -> top-K_c chunks -> ids/positions
// (+ optionally the token gather).
//
// PAPER.md sec:chunk_select: "we chunk the context contiguously and
// average the token score within each block, and then we select the Top-K
// blocks ... we apply a 1D average pooling before this"; sec:position_ids
// (P:125-133): kept tokens keep their original position ids; Alg.1
// merge_requests takes the selected tokens.
// Readings: shrinking pool edges (Z6), partial last chunk averaged
// over its true size (Z8), K_c from the exact ppm rule (Z9, computed on the
// host), ties to the lowest chunk index (Z10), ascending ids (Z11).
//
// Phase A can run on many CTAs per request (kModeA: grid (B, chunk blocks),
// writing cs to the workspace), phases B-C on one CTA of 1024 threads per
// request (kModeBC); short prompts run all three in one launch (kModeAll):
//   A. importance is staged in shared memory segment by segment (all loads of a
//      segment in flight together), pooled, and summed per chunk in token order
//      (deterministic) -> cs[c];
//   B. a 4-pass 8-bit radix select on the IEEE bits of cs (scores are >= 0, so
//      bit order == value order) finds the K_c-th largest value T; the digit
//      search is a parallel suffix scan over the 256 bins;
//   C. an in-order block scan keeps every chunk above T plus the lowest-index
//      chunks equal to T (exactly K_c chunks), compacts their token ranges into
//      ids/pos -- one warp per kept chunk, coalesced -- and, if requested,
//      gathers the kept tokens in the same pass.
#include "sp_internal.h"

#include <algorithm>

namespace sp {
namespace {

constexpr int ST = 1024;
constexpr int NW = ST / 32;
constexpr int SEG = 16384;          // tokens of importance staged in SMEM per segment (64 KiB)
constexpr int kMaxPool = 4097;      // largest pooling window (half-window staged on each side)
constexpr int kSmemChunks = 8192;   // chunk scores kept in SMEM when n_c fits (else L2-resident workspace)
enum SelectMode : int { kModeAll = 0, kModeA = 1, kModeBC = 2 };

struct ScanSmem {
  int warp_tot[NW];
  int total;
};

// Block-wide exclusive scan of v (all ST threads participate); returns the
// exclusive prefix, writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, ScanSmem& sm, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < NW ? sm.warp_tot[lane] : 0;
    int u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    if (lane < NW) sm.warp_tot[lane] = u - t;    // exclusive warp offsets
    if (lane == 31) sm.total = u;
  }
  __syncthreads();
  int res = sm.warp_tot[warp] + x - v;
  *total = sm.total;
  __syncthreads();                                 // sm reusable after return
  return res;
}

// Nrow: row length of the [B][Nrow] arrays; seq_lens (optional, row f3): the
// request's own prompt length n_b (clamped to [1, Nrow]), else Nrow.  K_c is
// computed per request from the keep rate in parts per million (Z9's integer rule).
__global__ void __launch_bounds__(ST) k_select(const float* __restrict__ imp_all, long long Nrow,
                                               const int* __restrict__ seq_lens, int pool_k, int chunk,
                                               int pos0, long long ppm, int* __restrict__ ids_all,
                                               int* __restrict__ pos_all, int* __restrict__ n_kept,
                                               float* __restrict__ cs_all, const int* __restrict__ tokens_all,
                                               int* __restrict__ out_all, int mode, int segcap, long long cpb) {
  extern __shared__ float seg[];                  // [segcap + 2w] staged importance, then [segcap] pooled
  __shared__ unsigned hist[256];
  __shared__ unsigned s_digit, s_remaining;
  __shared__ ScanSmem scan;
  __shared__ int kept_c[ST];                      // kept chunk ids of one scan tile, in order
  __shared__ int kept_off[ST];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long N = seq_lens ? std::min<long long>(std::max(seq_lens[b], 1), Nrow) : Nrow;
  const long long n_c = (N + chunk - 1) / chunk;
  const long long n_c_row = (Nrow + chunk - 1) / chunk;
  const long long K_c = std::min(n_c, std::max(1LL, (ppm * n_c + 999999) / 1000000));
  const float* imp = imp_all + (long long)b * Nrow;
  const long long w_ = (pool_k - 1) / 2;
  // chunk scores: SMEM when this CTA runs phases B-C and n_c fits, else the workspace
  // (decided on the row's chunk count, as the launch sized the SMEM: a ragged request may have fewer)
  const bool cs_smem = mode != kModeA && n_c_row <= kSmemChunks;
  float* cs = cs_smem ? seg + 2 * segcap + 2 * w_ : cs_all + (long long)b * n_c_row;
  int* ids = ids_all + (long long)b * Nrow;
  int* pos = pos_all + (long long)b * Nrow;
  const long long w = (pool_k - 1) / 2;

  if (mode == kModeBC) {
    if (cs_smem)
      for (long long c = tid; c < n_c; c += ST) cs[c] = cs_all[(long long)b * n_c_row + c];
    __syncthreads();
  } else {
  // ---- A. pooled scores (centred window, shrinking edges) -> chunk sums of
  //      chunks [c_lo, c_hi) (all of them unless kModeA)
  const long long c_lo = mode == kModeA ? std::min(n_c, (long long)blockIdx.y * cpb) : 0;
  const long long c_hi = mode == kModeA ? std::min(n_c, c_lo + cpb) : n_c;
  const long long t_lo = c_lo * chunk, t_hi = std::min(N, c_hi * chunk);
  float* pooled = seg + segcap + 2 * w;             // [segcap]
  const int wi = (int)w;
  const float inv_k = 1.f / (float)pool_k;
  const bool warp_chunks = chunk <= 32 && (chunk & (chunk - 1)) == 0;   // power of two <= 32
  for (long long base = t_lo; base < t_hi; base += segcap) {
    const int len = (int)((base + segcap < t_hi) ? segcap : t_hi - base);  // tokens in this segment
    const long long lo = base - w < 0 ? 0 : base - w, hi = base + len + w > N ? N : base + len + w;
    const int off = (int)(base - lo);                                     // seg index of token `base`
    {
      // all loads of the segment in flight before any store (latency-bound otherwise)
      constexpr int PER = SEG / ST;
      const int n = (int)(hi - lo);
      float r[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = tid + k * ST;
        r[k] = i < n ? __ldg(imp + lo + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = tid + k * ST;
        if (i < n) seg[i] = r[k];
      }
      for (int i = PER * ST + tid; i < n; i += ST) seg[i] = imp[lo + i];   // halo beyond SEG
    }
    __syncthreads();
    // interior tokens [i_lo, i_hi) have the full window inside the sequence
    const int i_lo = (int)(w - base > 0 ? w - base : 0);
    const int i_hi = (int)(N - 1 - w - base + 1 < len ? N - 1 - w - base + 1 : len);
#pragma unroll 4
    for (int i = tid; i < len; i += ST) {                               // coalesced, conflict-free
      float ws = 0.f;
      if (i >= i_lo && i < i_hi) {                                      // interior: full window
        const float* p0 = seg + off + i - wi;
        for (int k = 0; k < pool_k; ++k) ws += p0[k];
        pooled[i] = ws * inv_k;
      } else {                                                            // sequence edges: shrink
        const long long t = base + i;
        const long long a = t - w < 0 ? 0 : t - w, e = t + w > N - 1 ? N - 1 : t + w;
        for (long long j = a; j <= e; ++j) ws += seg[j - lo];
        pooled[i] = ws / (float)(e - a + 1);
      }
    }
    __syncthreads();
    const long long c_first = base / chunk, c_last = (base + len - 1) / chunk;
    if (warp_chunks && base % chunk == 0) {
      // a warp sums 32 consecutive pooled values in groups of `chunk` lanes (tree
      // order); segcap is a multiple of 32 so every chunk starts inside its segment
      const int lg = __ffs(chunk) - 1;
      const int cbase = (int)(base >> lg);
#pragma unroll 4
      for (int g0 = warp * 32; g0 < len; g0 += ST) {
        float v = g0 + lane < len ? pooled[g0 + lane] : 0.f;
        for (int o = chunk >> 1; o >= 1; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, chunk);
        if ((lane & (chunk - 1)) == 0 && g0 + lane < len) cs[cbase + ((g0 + lane) >> lg)] = v;
      }
    } else {
      // the owner thread walks its chunk's tokens in a rotated (fixed, hence
      // deterministic) order so a warp's reads hit distinct banks
      for (long long c = c_first + tid; c <= c_last; c += ST) {
        const long long t0 = c * chunk > base ? c * chunk : base;
        const long long t1 = (c + 1) * chunk < base + len ? (c + 1) * chunk : base + len;
        const int n = (int)(t1 - t0), i0 = (int)(t0 - base);
        float sacc = (t0 == c * chunk) ? 0.f : cs[c];                    // chunk continued from the previous segment
        const int rot = (int)(c % n);
        for (int j = 0; j < n; ++j) {
          int k = j + rot;
          if (k >= n) k -= n;
          sacc += pooled[i0 + k];
        }
        cs[c] = sacc;
      }
    }
    __syncthreads();
  }
  for (long long c = c_lo + tid; c < c_hi; c += ST) {
    const long long sz = ((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk;
    cs[c] = cs[c] / (float)sz;
  }
  __syncthreads();
  }
  if (mode == kModeA) return;

  // ---- B. radix select: threshold bit pattern T of the K_c-th largest score.
  //      Up to kRankMax chunks the rank is counted directly instead:
  //      rank(c) = #{c' : cs[c'] > cs[c], or cs[c'] == cs[c] and c' < c} (the
  //      (score desc, index asc) order), kept iff rank < K_c -- one pass, no
  //      barrier rounds (measured: 2 us faster at 128 chunks, 29 us slower at 1024).
  constexpr int kRankMax = 256;
  const bool by_rank = n_c <= kRankMax;
  unsigned prefix = 0, pmask = 0;
  unsigned remaining = (unsigned)K_c;
  int rank_keep = 0;
  if (by_rank) {
    if (tid < n_c) {
      const float mine = cs[tid];
      int rank = 0;
#pragma unroll 8
      for (int c2 = 0; c2 < (int)n_c; ++c2) {
        const float o = cs[c2];                      // same address in every lane: broadcast
        rank += (o > mine || (o == mine && c2 < tid)) ? 1 : 0;
      }
      rank_keep = rank < K_c ? 1 : 0;
    }
  }
  for (int shift = 24; shift >= 0 && !by_rank; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    // warp-aggregated: lanes with the same digit add once (the top digits of
    // near-equal scores collide, and SMEM atomics on one address serialise)
    for (long long c0 = (long long)warp * 32; c0 < n_c; c0 += ST) {
      const long long c = c0 + lane;
      const unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
      const unsigned digit = (c < n_c && (key & pmask) == prefix) ? (key >> shift) & 255u : 256u;
      const unsigned peers = __match_any_sync(0xffffffffu, digit);
      if (digit < 256u && lane == __ffs(peers) - 1) atomicAdd(&hist[digit], (unsigned)__popc(peers));
    }
    __syncthreads();
    // digit D: count(digits > D) < remaining <= count(digits >= D); warps 0-7 scan 256 bins
    if (tid < 256) {
      // suffix sums over bins (high digit first): bin d handled by thread 255 - d
      const int d = 255 - tid;
      unsigned v = hist[d];
      unsigned x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) scan.warp_tot[warp] = (int)x;
      __syncwarp();
      // (warps 0..7 only) combine warp totals below
      kept_off[tid] = (int)x;                      // inclusive within warp
    }
    __syncthreads();
    if (tid < 256) {
      unsigned before = 0;
      for (int ww = 0; ww < warp; ++ww) before += (unsigned)scan.warp_tot[ww];
      const unsigned incl = before + (unsigned)kept_off[tid];   // count of digits >= d
      const unsigned excl = incl - hist[255 - tid];             // count of digits > d
      if (excl < remaining && incl >= remaining) {
        s_digit = (unsigned)(255 - tid);
        s_remaining = remaining - excl;
      }
    }
    __syncthreads();
    prefix |= s_digit << shift;
    pmask |= 255u << shift;
    remaining = s_remaining;
    __syncthreads();
  }
  const unsigned T = prefix;
  const int need_eq = (int)remaining;            // chunks equal to T to keep (lowest indices first)

  // ---- C. keep flags in chunk order, compaction (+ gather) of the kept token ranges
  int carry_eq = 0, carry_tok = 0;
  const int* tokens = tokens_all ? tokens_all + (long long)b * Nrow : nullptr;
  int* out = out_all ? out_all + (long long)b * Nrow : nullptr;
  for (long long base = 0; base < n_c; base += ST) {
    const long long c = base + tid;
    const unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
    const int eq = (c < n_c && key == T) ? 1 : 0;
    const int gt = (c < n_c && key > T) ? 1 : 0;
    int tot;
    const int eq_rank = block_excl_scan(eq, scan, &tot) + carry_eq;
    carry_eq += tot;
    const int keep = by_rank ? rank_keep : (gt | (eq & (eq_rank < need_eq ? 1 : 0)));
    const int slot = block_excl_scan(keep, scan, &tot);          // index among kept chunks of this tile
    const int nk = tot;
    int sz = 0;
    if (keep) sz = (int)(((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk);
    int tot2;
    const int off = block_excl_scan(sz, scan, &tot2) + carry_tok;
    if (keep) {
      kept_c[slot] = (int)c;
      kept_off[slot] = off;
    }
    __syncthreads();
    // one warp per kept chunk: coalesced ids / pos (/ gathered tokens)
    for (int k = warp; k < nk; k += NW) {
      const long long cc = kept_c[k];
      const int t0 = (int)(cc * chunk);
      const int csz = (int)(((cc + 1) * chunk < N ? (cc + 1) * chunk : N) - cc * chunk);
      const int o = kept_off[k];
      for (int j = lane; j < csz; j += 32) {
        ids[o + j] = t0 + j;
        pos[o + j] = t0 + j + pos0;
        if (out) out[o + j] = tokens[t0 + j];
      }
    }
    carry_tok += tot2;
    __syncthreads();
  }
  if (tid == 0) n_kept[b] = carry_tok;
}

}  // namespace

size_t select_ws_bytes(int B, long long N, int chunk) {
  long long n_c = (N + chunk - 1) / chunk;
  return align256((size_t)B * n_c * sizeof(float));
}

bool select_supported(int pool_k) { return pool_k <= kMaxPool; }

cudaError_t select_launch(const float* imp, int B, long long N, int pool_k, int chunk, int pos0, long long ppm,
                          int* ids, int* pos, int* n_kept, void* ws, cudaStream_t st, const int* tokens, int* out,
                          const int* seq_lens) {
  static bool configured = false;
  const size_t smem_max = (size_t)(2 * SEG + 2 * ((kMaxPool - 1) / 2) + kSmemChunks) * sizeof(float);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long long n_c = (N + chunk - 1) / chunk;
  const long long w = (pool_k - 1) / 2;
  float* cs = reinterpret_cast<float*>(ws);
  // Long prompts: phase A (pooling + chunk sums, the bulk of the work) on
  // ~kTokPerCta-token blocks of chunks spread over the SMs, then B-C per request.
  constexpr long long kTokPerCta = 2048;
  const long long cpb = std::max(1LL, kTokPerCta / chunk);
  const long long nblk = (n_c + cpb - 1) / cpb;
  if (nblk >= 4 && nblk <= 65535) {
    const long long span = std::min(N, cpb * chunk);
    const int segcap = (int)std::min<long long>(SEG, (span + 31) / 32 * 32);
    const size_t needA = (size_t)(2 * segcap + 2 * w) * sizeof(float);
    k_select<<<dim3(B, (unsigned)nblk), ST, needA, st>>>(imp, N, seq_lens, pool_k, chunk, pos0, ppm, ids, pos, n_kept, cs, tokens,
                                                        out, kModeA, segcap, cpb);
    const size_t needBC = (size_t)(2 * segcap + 2 * w + (n_c <= kSmemChunks ? n_c : 0)) * sizeof(float);
    k_select<<<B, ST, needBC, st>>>(imp, N, seq_lens, pool_k, chunk, pos0, ppm, ids, pos, n_kept, cs, tokens, out, kModeBC,
                                    segcap, cpb);
    return cudaGetLastError();
  }
  const size_t need = (size_t)(2 * SEG + 2 * w + (n_c <= kSmemChunks ? n_c : 0)) * sizeof(float);
  k_select<<<B, ST, need, st>>>(imp, N, seq_lens, pool_k, chunk, pos0, ppm, ids, pos, n_kept, cs, tokens, out, kModeAll, SEG,
                                n_c);
  return cudaGetLastError();
}

}  // namespace sp
