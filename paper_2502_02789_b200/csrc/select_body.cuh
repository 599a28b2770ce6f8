// The selection kernel's body (select.cu), as a device function over NT
// threads, so that the standalone kernel (NT = 1024) and the score kernel's
// fused tail (NT = 384, score_fused.cu) run the same code and give the same
// bits.  See select.cu for the method and its citations.  Internal header.
#pragma once

#include <math_constants.h>

#include <algorithm>

#include "sp_internal.h"

namespace sp {
namespace sel {

constexpr int SEG = 16384;          // tokens of importance staged in SMEM per segment (64 KiB)
constexpr int kMaxPool = 4097;      // largest pooling window (half-window staged on each side)
constexpr int kSmemChunks = 8192;   // chunk scores kept in SMEM when n_c fits (else L2-resident workspace)
constexpr unsigned kInvalid = 0xFFFFFFFFu;   // merge: chunk with no candidate (never a score: scores are >= 0)
enum SelectMode : int { kModeAll = 0, kModeA = 1 };
enum Variant : int { kPlain = 0, kCand = 1, kMerge = 2 };

// Debug timeline (-DSP_SELECT_TRACE builds only, tools/sel_trace.py): globaltimer
// stamps of the selection's phases in g_sel_trace (select.cu).
#ifdef SP_SELECT_TRACE
__device__ unsigned long long g_sel_trace[16];   // (select.cu is the only includer)
#define SEL_STAMP(k) \
  do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
       g_sel_trace[k] = t_; } } while (0)
#define SEL_STAMP_MIN(k) \
  do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
       atomicMin(&g_sel_trace[k], t_); } } while (0)
#else
#define SEL_STAMP(k) do { } while (0)
#define SEL_STAMP_MIN(k) do { } while (0)
#endif

struct SelArgs {
  const float* imp;          // [B][row] importance (kCand: this rank's shard)
  int nreq;                  // B (rows of every [B][...] array)
  int nblk;                  // kModeA: phase-A blocks per request
  int sh_off;                // floats from the dynamic SMEM base to the SelShared scratch
  unsigned* blk_cnt;         // [B] kModeA: phase-A CTAs done (workspace, zero, self-resetting)
  long long row;             // row length of imp / ids / pos / tokens / out
  const int* seq_lens;       // kPlain, optional [B]: per-request prompt length (row f3)
  int pool_k, chunk, pos0;
  long long ppm;             // keep rate in parts per million (K_c, Z9)
  int* ids;
  int* pos;
  int* n_kept;
  float* cs_ws;              // [B][n_c_row] chunk scores (workspace)
  const int* tokens;         // optional gather source [B][row]
  int* out;                  // optional gathered tokens [B][row]
  int mode, segcap;
  // kPlain, deferred finalize (sp_score_select): the importance is not written
  // by the score kernel; phase A computes it from the unit groups' partial
  // (l,h)-max maps, imp[t] = (1/Rv) sum_r 2^(max_g accp[b][g][r][t]) -- the
  // score kernel's own finalize, same instruction, same order -- and writes it
  const float* accp;         // [B][n_ug][Rv][acc_pitch], or null
  long long acc_pitch;
  int n_ug, Rv;
  float* imp_out;            // [B][row]
  int mb_off;                // floats from the dynamic SMEM base to the [Rv][segcap + 2w] max scratch
  int cs_ready;              // kPlain: the chunk scores are already in cs_ws (computed by the score
                             // kernel's epilogue, sp_score_select): phases B-C only
  long long cpb;             // chunks per CTA in kModeA
  // sequence sharding
  long long i0;              // kCand: global index of this shard's first token
  long long n_glob;          // kCand / kMerge: prompt length N (kPlain: row / seq_lens)
  const float* edges;        // kCand: [P][B][2w] first w / last w importance values of every rank
  int rank, world;
  long long k_sel;           // kCand: M
  unsigned long long* cand;  // kCand: [B][M] candidate keys out
  const unsigned long long* cand_in;   // kMerge: [P][B][M] candidate keys
};

template <int NT>
struct ScanSmem {
  int warp_tot[NT / 32];
  int total;
  unsigned long long warp_tot64[NT / 32];
  unsigned long long total64;
};

// The selection's shared scratch (besides the staged importance / chunk scores),
// for NT threads: placed in dynamic shared memory by the caller.
template <int NT>
struct SelShared {
  unsigned hist[4 * 256];           // one histogram per radix pass (zeroed together: one barrier per pass)
  unsigned s_digit, s_remaining;
  int s_last;
  ScanSmem<NT> scan;
  int kept_c[NT];                   // kept chunk ids of one scan tile, in order
  int kept_off[NT];
};

// 2^x as the score kernel computes it (ex2.approx.ftz.f32): the deferred
// finalize gives the importance bit for bit.
__device__ __forceinline__ float sel_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Block-wide exclusive scan of v (all NT threads participate); returns the
// exclusive prefix, writes the block total to *total.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, ScanSmem<NT>& sm, int* total) {
  constexpr int NW = NT / 32;
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

// The same over 64-bit values (two packed counters: kept chunks << 32 | kept tokens).
template <int NT>
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v, ScanSmem<NT>& sm,
                                                                unsigned long long* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.warp_tot64[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long t = lane < NW ? sm.warp_tot64[lane] : 0ull;
    unsigned long long u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    if (lane < NW) sm.warp_tot64[lane] = u - t;
    if (lane == 31) sm.total64 = u;
  }
  __syncthreads();
  const unsigned long long res = sm.warp_tot64[warp] + x - v;
  *total = sm.total64;
  return res;                                      // (callers barrier before reusing sm)
}

// Segment length starting at chunk-aligned token `base`: whole chunks when a
// chunk fits the segment, else the rest of the chunk up to segcap tokens.
__device__ __forceinline__ long long seg_len(long long base, long long t_hi, int chunk, int segcap) {
  long long next;
  if (chunk <= segcap) {
    next = base + (long long)(segcap / chunk) * chunk;
  } else {
    const long long cend = (base / chunk + 1) * chunk;
    next = base + segcap < cend ? base + segcap : cend;
  }
  return (next < t_hi ? next : t_hi) - base;
}


// One CTA's share of the selection of request b: phase A over chunk block blk
// (kModeA) or all three phases (kModeAll); in kModeA the request's last block
// to finish continues with B-C.  seg: dynamic shared memory of
// (2 segcap + 2w + (n_c if it fits)) floats; sh: the shared scratch.
template <int V, int NT>
__device__ __forceinline__ void select_body(const SelArgs& a, int b, int blk, float* seg, SelShared<NT>& sh) {
  const int mode = a.mode, chunk = a.chunk, pool_k = a.pool_k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long Nrow = a.row;
  // N: the prompt length the pooling edges and chunk sizes refer to (global when sharded)
  long long N;
  if (V == kPlain) N = a.seq_lens ? std::min<long long>(std::max(a.seq_lens[b], 1), Nrow) : Nrow;
  else N = a.n_glob;
  const long long i0 = V == kCand ? a.i0 : 0;                    // global index of imp[b][0]
  const long long n_loc = V == kCand ? Nrow : N;                 // tokens held in imp rows
  const long long c_base = i0 / chunk;                           // global id of local chunk 0
  const long long n_c_all = (N + chunk - 1) / chunk;             // chunks of the prompt
  const long long n_c = V == kCand ? n_loc / chunk : n_c_all;    // chunks this selection ranks
  const long long n_c_row = V == kPlain ? (Nrow + chunk - 1) / chunk : n_c;   // workspace row
  long long K_sel;
  if (V == kCand) K_sel = a.k_sel;
  else K_sel = std::min(n_c_all, std::max(1LL, (a.ppm * n_c_all + 999999) / 1000000));
  const float* imp = a.imp + (long long)b * Nrow;
  const long long w = (pool_k - 1) / 2;
  // chunk scores: SMEM when this CTA runs phases B-C and n_c fits, else the workspace
  // (decided on the row's chunk count, as the launch sized the SMEM: a ragged request may have fewer)
  const bool cs_smem = mode == kModeAll && n_c_row <= kSmemChunks;
  float* cs = cs_smem ? seg + 2 * a.segcap + 2 * w : a.cs_ws + (long long)b * n_c_row;

  if (V == kPlain && a.cs_ready) {
    // ---- the chunk scores were computed by the score kernel (same arithmetic, same bits)
    if (cs_smem) {
      const float* src = a.cs_ws + (long long)b * n_c_row;
      for (long long c = tid; c < n_c; c += NT) cs[c] = __ldcg(src + c);
    } else {
      cs = a.cs_ws + (long long)b * n_c_row;
    }
    __syncthreads();
  } else if (V == kMerge) {
    // ---- scatter the P ranks' candidates into the dense chunk array
    unsigned* csu = reinterpret_cast<unsigned*>(cs);
    for (long long c = tid; c < n_c; c += NT) csu[c] = kInvalid;
    __syncthreads();
    const long long M = a.k_sel;
    for (int p = 0; p < a.world; ++p) {
      const unsigned long long* src = a.cand_in + ((long long)p * a.nreq + b) * M;
      for (long long m = tid; m < M; m += NT) {
        const unsigned long long key = src[m];
        const unsigned c = ~(unsigned)(key & 0xFFFFFFFFull);
        if (c < (unsigned long long)n_c) csu[c] = (unsigned)(key >> 32);
      }
    }
    __syncthreads();
  } else {
  // ---- A. pooled scores (centred window, shrinking edges) -> chunk sums of
  //      chunks [c_lo, c_hi) (global ids; all of the CTA's range unless kModeA)
  const long long c_lo = c_base + (mode == kModeA ? std::min(n_c, (long long)blk * a.cpb) : 0);
  const long long c_hi = c_base + (mode == kModeA ? std::min(n_c, (long long)blk * a.cpb + a.cpb) : n_c);
  const long long t_lo = c_lo * chunk, t_hi = std::min(N, c_hi * chunk);
  const int segcap = a.segcap;
  float* pooled = seg + segcap + 2 * w;             // [segcap]
  const int wi = (int)w;
  const float inv_k = 1.f / (float)pool_k;
  const bool warp_chunks = chunk <= 32 && (chunk & (chunk - 1)) == 0;   // power of two <= 32
  // kCand: importance of global token t in [i0 - w, i0 + n_loc + w): own shard, or a neighbour's edge
  const float* halo_l = nullptr;
  const float* halo_r = nullptr;
  if (V == kCand) {
    const long long eb = 2 * w;                       // edges row: first w, then last w values
    if (a.rank > 0) halo_l = a.edges + ((long long)(a.rank - 1) * a.nreq + b) * eb + w;
    if (a.rank + 1 < a.world) halo_r = a.edges + ((long long)(a.rank + 1) * a.nreq + b) * eb;
  }
  for (long long base = t_lo; base < t_hi;) {
    const int len = (int)seg_len(base, t_hi, chunk, segcap);             // tokens in this segment
    const long long lo = base - w < 0 ? 0 : base - w, hi = base + len + w > N ? N : base + len + w;
    const int off = (int)(base - lo);                                     // seg index of token `base`
    {
      // all loads of the segment in flight before any store (latency-bound otherwise)
      constexpr int PER = (SEG / NT) < 16 ? (SEG / NT) : 16;
      const int n = (int)(hi - lo);
      float r[PER];
      if (V == kPlain && a.accp != nullptr) {
        // deferred finalize: every (group, row, token) value of the staged range
        // loaded with all of a thread's loads in flight (coalesced over tokens)
        // and folded into SMEM with an order-preserving unsigned max (order-free:
        // the same bits as a sequential max), then one thread per token takes
        // the mean of exp2 in row order; the CTA's own tokens' importance is
        // written out
        const int n = (int)(hi - lo), Rv = a.Rv, RN = Rv * n, tot = a.n_ug * RN;
        unsigned* mb = reinterpret_cast<unsigned*>(seg + a.mb_off);   // [Rv][n]
        for (int e = tid; e < RN; e += NT) mb[e] = 0u;                  // below every ordered key
        __syncthreads();
        const float* src = a.accp + (long long)b * a.n_ug * Rv * a.acc_pitch + lo;
        // element e = q*n + j (q = group*Rv + row), e = tid + k*NT: the indices
        // advance by a fixed (dq, dj) per step (no per-element division)
        const int dq = NT / n, dj = NT - dq * n, dr = dq % Rv;
        int q = tid / n, j = tid - q * n, r = q % Rv;
        const long long pitch = a.acc_pitch, step = (long long)dq * pitch + dj, wrap = pitch - n;
        const float* ptr = src + (long long)q * pitch + j;
        for (int e0 = tid; e0 < tot; e0 += 16 * NT) {
          float v[16];
          int dst[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const bool in = e0 + k * NT < tot;
            dst[k] = in ? r * n + j : -1;
            v[k] = __ldcg(in ? ptr : src);                          // (branch-free: src is a valid address)
            j += dj;
            r += dr;
            ptr += step;
            if (j >= n) { j -= n; ++r; ptr += wrap; }
            if (r >= Rv) r -= Rv;
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            if (dst[k] >= 0) {
              const unsigned u = __float_as_uint(v[k]);
              atomicMax(&mb[dst[k]], (u & 0x80000000u) ? ~u : (u | 0x80000000u));
            }
          }
        }
        __syncthreads();
        const float inv = 1.f / (float)Rv;
        for (int j = tid; j < n; j += NT) {
          float sacc = 0.f;
          for (int r = 0; r < Rv; ++r) {
            const unsigned k = mb[r * n + j];
            sacc += sel_ex2(__uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k));
          }
          const float v = sacc * inv;
          seg[j] = v;
          const long long t = lo + j;
          if (t >= t_lo && t < t_hi) a.imp_out[(long long)b * Nrow + t] = v;
        }
      } else if (V == kCand) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = tid + k * NT;
          const long long t = lo + i;
          r[k] = i >= n ? 0.f
                        : (t < i0 ? __ldcg(halo_l + (t - (i0 - w)))
                                  : (t >= i0 + n_loc ? __ldcg(halo_r + (t - i0 - n_loc)) : __ldcg(imp + (t - i0))));
        }
      } else {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = tid + k * NT;
          r[k] = i < n ? __ldcg(imp + lo + i) : 0.f;
        }
      }
      if (!(V == kPlain && a.accp != nullptr)) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = tid + k * NT;
          if (i < n) seg[i] = r[k];
        }
        for (int i = PER * NT + tid; i < n; i += NT) {                  // halo beyond SEG
          const long long t = lo + i;
          if (V == kCand)
            seg[i] = t < i0 ? halo_l[t - (i0 - w)] : (t >= i0 + n_loc ? halo_r[t - i0 - n_loc] : imp[t - i0]);
          else
            seg[i] = imp[t];
        }
      }
    }
    __syncthreads();
    SEL_STAMP(6);
    // interior tokens [i_lo, i_hi) have the full window inside the sequence
    const int i_lo = (int)(w - base > 0 ? w - base : 0);
    const int i_hi = (int)(N - 1 - w - base + 1 < len ? N - 1 - w - base + 1 : len);
#pragma unroll 4
    for (int i = tid; i < len; i += NT) {                               // coalesced, conflict-free
      float ws = 0.f;
      if (i >= i_lo && i < i_hi) {                                      // interior: full window
        const float* p0 = seg + off + i - wi;
        for (int k = 0; k < pool_k; ++k) ws += p0[k];
        pooled[i] = ws * inv_k;
      } else {                                                            // sequence edges: shrink
        const long long t = base + i;
        const long long e0 = t - w < 0 ? 0 : t - w, e1 = t + w > N - 1 ? N - 1 : t + w;
        for (long long j = e0; j <= e1; ++j) ws += seg[j - lo];
        pooled[i] = ws / (float)(e1 - e0 + 1);
      }
    }
    __syncthreads();
    SEL_STAMP(7);
    const long long c_first = base / chunk, c_last = (base + len - 1) / chunk;
    if (warp_chunks) {
      // a warp sums 32 consecutive pooled values in groups of `chunk` lanes (tree
      // order); segments start on chunk boundaries and hold whole chunks
      const int lg = __ffs(chunk) - 1;
      const long long cb = (base >> lg) - c_base;
#pragma unroll 4
      for (int g0 = warp * 32; g0 < len; g0 += NT) {
        float v = g0 + lane < len ? pooled[g0 + lane] : 0.f;
        for (int o = chunk >> 1; o >= 1; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, chunk);
        if ((lane & (chunk - 1)) == 0 && g0 + lane < len) cs[cb + ((g0 + lane) >> lg)] = v;
      }
    } else {
      // the owner thread walks its chunk's tokens in a rotated (fixed, hence
      // deterministic) order so a warp's reads hit distinct banks
      for (long long c = c_first + tid; c <= c_last; c += NT) {
        const long long t0 = c * chunk > base ? c * chunk : base;
        const long long t1 = (c + 1) * chunk < base + len ? (c + 1) * chunk : base + len;
        const int n = (int)(t1 - t0), ii = (int)(t0 - base);
        float sacc = (t0 == c * chunk) ? 0.f : cs[c - c_base];          // chunk continued from the previous segment
        const int rot = (int)(c % n);
        for (int j = 0; j < n; ++j) {
          int k = j + rot;
          if (k >= n) k -= n;
          sacc += pooled[ii + k];
        }
        cs[c - c_base] = sacc;
      }
    }
    __syncthreads();
    SEL_STAMP(8);
    base += len;
  }
  for (long long c = c_lo + tid; c < c_hi; c += NT) {
    const long long sz = ((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk;
    cs[c - c_base] = cs[c - c_base] / (float)sz;
  }
  __syncthreads();
  }
  SEL_STAMP(2);
  if (mode == kModeA) {
    // the request's last phase-A CTA to finish runs phases B-C (one launch for
    // the whole selection): every CTA publishes its chunk scores, then counts
    __threadfence();
    __syncthreads();
    if (tid == 0) sh.s_last = atomicAdd(a.blk_cnt + b, 1u) + 1u == a.nblk;
    __syncthreads();
    if (!sh.s_last) return;
    __threadfence();
    if (tid == 0) a.blk_cnt[b] = 0u;                                     // self-resetting for the next call
    if (n_c_row <= kSmemChunks) {                                       // the launch sized SMEM for it
      float* cs_s = seg + 2 * a.segcap + 2 * w;
      for (long long c = tid; c < n_c; c += NT) cs_s[c] = __ldcg(cs + c);
      cs = cs_s;
    }
    __syncthreads();
  }
  SEL_STAMP(3);

  // ---- B. radix select: threshold T of the K_sel-th largest score, as a bit
  //      prefix (T & pmask): a chunk is above the threshold iff (key & pmask) >
  //      prefix, at it iff equal.  4 passes of 8 bits over the IEEE bits (scores
  //      are >= 0, so bit order == value order), each pass one histogram and ONE
  //      barrier: every warp then finds the digit itself from the 256 bins (no
  //      second barrier round); a pass whose threshold bin holds exactly the
  //      chunks still needed ends the search (all of them are kept).
  //      Up to kRankMax chunks the rank is counted directly instead:
  //      rank(c) = #{c' : cs[c'] > cs[c], or cs[c'] == cs[c] and c' < c} (the
  //      (score desc, index asc) order), kept iff rank < K_sel, by S threads per
  //      chunk (strided subsets, shuffle-summed).
  //      kMerge: invalid entries (bit pattern kInvalid, a NaN) never count.
  constexpr int kRankMax = 256;
  const bool by_rank = n_c <= kRankMax && n_c <= NT;
  unsigned prefix = 0, pmask = 0;
  unsigned remaining = (unsigned)K_sel;
  unsigned eq_total = 0;                             // chunks at the threshold (its bin in the last pass)
  if (by_rank) {
    int lg = 0;
    while (lg < 5 && ((long long)NT >> (lg + 1)) >= n_c) ++lg;   // S = 2^lg threads per chunk, S * n_c <= NT
    const int S = 1 << lg;
    const int c = tid >> lg, part = tid & (S - 1);
    int rank = 0;
    float mine = 0.f;
    if (c < n_c) {
      mine = cs[c];
#pragma unroll 8
      for (int c2 = part; c2 < (int)n_c; c2 += S) {
        const float o = cs[c2];                      // same address in every lane of a group: broadcast
        rank += (o > mine || (o == mine && c2 < c)) ? 1 : 0;
      }
    }
    for (int o = 1; o < S; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (part == 0 && c < n_c) {
      int keep = rank < K_sel ? 1 : 0;
      if (V == kMerge && __float_as_uint(mine) == kInvalid) keep = 0;
      sh.kept_off[c] = keep;                         // keep flags by chunk (phase C reads them)
    }
    __syncthreads();
  } else {
    for (int i = tid; i < 4 * 256; i += NT) sh.hist[i] = 0u;
    __syncthreads();
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      unsigned* H = sh.hist + 256 * pass;
      // a warp whose lanes share one digit (the top digits of near-equal
      // scores: SMEM atomics on one address serialise) adds once; otherwise
      // every lane adds its own
      if (n_c <= 4 * NT) {
        for (long long c0 = (long long)warp * 32; c0 < n_c; c0 += NT) {
          const long long c = c0 + lane;
          const unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
          const bool in = c < n_c && (V != kMerge || key != kInvalid);
          const unsigned digit = (in && (key & pmask) == prefix) ? (key >> shift) & 255u : 256u;
          const unsigned d0 = __shfl_sync(0xffffffffu, digit, 0);
          if (__all_sync(0xffffffffu, digit == d0)) {
            if (lane == 0 && d0 < 256u) atomicAdd(&H[d0], 32u);
          } else if (digit < 256u) {
            atomicAdd(&H[digit], 1u);
          }
        }
      } else {
        constexpr int U = 8;                                     // keys in flight per lane (latency-bound otherwise)
        for (long long c0 = (long long)warp * 32; c0 < n_c; c0 += (long long)NT * U) {
          unsigned keys[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long long c = c0 + (long long)u * NT + lane;
            keys[u] = c < n_c ? __float_as_uint(cs[c]) : kInvalid;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long long c = c0 + (long long)u * NT + lane;
            const bool in = c < n_c && (V != kMerge || keys[u] != kInvalid);
            const unsigned digit = (in && (keys[u] & pmask) == prefix) ? (keys[u] >> shift) & 255u : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, digit);
            if (digit < 256u && lane == __ffs(peers) - 1) atomicAdd(&H[digit], (unsigned)__popc(peers));
          }
        }
      }
      __syncthreads();
      // digit D: count(digits > D) < remaining <= count(digits >= D).  Every warp
      // scans the 256 bins itself: lane l holds digits 255 - 8l - k, k = 0..7.
      const uint4 lo4 = *reinterpret_cast<const uint4*>(H + 248 - 8 * lane);
      const uint4 hi4 = *reinterpret_cast<const uint4*>(H + 252 - 8 * lane);
      const unsigned cnt[8] = {hi4.w, hi4.z, hi4.y, hi4.x, lo4.w, lo4.z, lo4.y, lo4.x};
      unsigned t = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += cnt[k];
      unsigned incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - t;
      const bool here = excl < remaining && incl >= remaining;
      const unsigned ball = __ballot_sync(0xffffffffu, here);
      unsigned dig = 0, before = 0, bin = 0;
      if (here) {
        unsigned run = excl;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (bin == 0u && run + cnt[k] >= remaining) {
            dig = 255u - 8u * lane - k;
            before = run;
            bin = cnt[k];
          }
          run += cnt[k];
        }
      }
      const int src = ball ? __ffs(ball) - 1 : 0;
      dig = __shfl_sync(0xffffffffu, dig, src);
      before = __shfl_sync(0xffffffffu, before, src);
      bin = __shfl_sync(0xffffffffu, bin, src);
      prefix |= dig << shift;
      pmask |= 255u << shift;
      remaining -= before;
      eq_total = bin;
      SEL_STAMP(10 + pass);
      if (bin == remaining) break;                   // every chunk of the threshold bin is kept
    }
  }
  SEL_STAMP(4);
  const unsigned T = prefix;
  const int need_eq = (int)remaining;            // chunks at the threshold to keep (lowest indices first)

  // ---- C. keep flags in chunk order, compaction (+ gather) of the kept token
  //      ranges, or (kCand) the kept chunks' candidate keys
  int carry_eq = 0, carry_tok = 0, carry_k = 0;
  const int* tokens = a.tokens ? a.tokens + (long long)b * Nrow : nullptr;
  int* out = a.out ? a.out + (long long)b * Nrow : nullptr;
  int* ids = V == kCand ? nullptr : a.ids + (long long)b * Nrow;
  int* pos = V == kCand ? nullptr : a.pos + (long long)b * Nrow;
  if (n_c <= NT) {
    // one tile of chunks (every prompt up to NT chunks): thread c owns chunk c.
    // The tie scan only when the threshold has more chunks than are kept; one
    // packed scan gives each kept chunk its slot and its first output token;
    // then a flat compaction: kept token o lies in kept chunk o / chunk (only the
    // prompt's last chunk can be short, and it is the last kept one), so the
    // token gather's loads are independent (no per-chunk chain).
    const int c = tid;
    const unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
    const bool in = c < n_c && (V != kMerge || key != kInvalid);
    int keep;
    if (by_rank) {
      keep = c < n_c ? sh.kept_off[c] : 0;
    } else {
      const int eq = (in && (key & pmask) == T) ? 1 : 0;
      const int gt = (in && (key & pmask) > T) ? 1 : 0;
      if ((int)eq_total == need_eq) {
        keep = gt | eq;
      } else {
        int tot;
        const int eq_rank = block_excl_scan<NT>(eq, sh.scan, &tot);
        keep = gt | (eq & (eq_rank < need_eq ? 1 : 0));
      }
    }
    __syncthreads();                                  // (kept_off / scan scratch reused below)
    if (V == kCand) {
      int tot;
      const int slot = block_excl_scan<NT>(keep, sh.scan, &tot);
      if (keep)
        a.cand[(long long)b * K_sel + slot] = ((unsigned long long)key << 32) | (unsigned long long)(~(unsigned)(c + c_base));
      return;
    }
    const int sz = keep ? (int)(((long long)(c + 1) * chunk < N ? (long long)(c + 1) * chunk : N) - (long long)c * chunk) : 0;
    unsigned long long tot2;
    const unsigned long long pk = block_excl_scan64<NT>(((unsigned long long)keep << 32) | (unsigned)sz, sh.scan, &tot2);
    if (keep) sh.kept_c[(int)(pk >> 32)] = c;
    const int n_tok = (int)(tot2 & 0xFFFFFFFFull);
    __syncthreads();
#pragma unroll 4
    for (int o = tid; o < n_tok; o += NT) {
      const int s2 = o / chunk;
      const int t = sh.kept_c[s2] * chunk + (o - s2 * chunk);
      ids[o] = t;
      pos[o] = t + a.pos0;
      if (out) out[o] = tokens[t];
    }
    if (tid == 0) a.n_kept[b] = n_tok;
    SEL_STAMP(5);
    return;
  }
  if (n_c > 4 * NT && !by_rank) {
    // many chunks (token-level selection of long prompts): every warp owns a
    // contiguous range of chunks and walks it in coalesced 32-chunk tiles
    // (ballots / shuffles inside the warp), so the block needs three scans in
    // all instead of three per NT-chunk tile; the same keep rule (every chunk
    // above T, the lowest-index chunks equal to T) and the same output order
    constexpr int NWP = NT / 32;
    const long long per = ((n_c + NWP - 1) / NWP + 31) / 32 * 32;
    const long long w0 = std::min(n_c, (long long)warp * per), w1 = std::min(n_c, w0 + per);
    const unsigned lt = (1u << lane) - 1u;
    auto flags_of = [&](long long c, unsigned key, bool* eq, bool* gt) {
      const bool in = c < w1 && (V != kMerge || key != kInvalid);
      *eq = in && (key & pmask) == T;
      *gt = in && (key & pmask) > T;
    };
    constexpr int TU = 4;                                    // tiles whose keys are loaded together
    auto load4 = [&](long long c0, unsigned (&k4)[TU]) {
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const long long c = c0 + 32 * u + lane;
        k4[u] = c < w1 ? __float_as_uint(cs[c]) : 0u;                    // (SMEM or workspace)
      }
    };
    auto csize = [&](long long c) { return (int)(((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk); };
    int w_eq = 0;
    for (long long c1 = w0; c1 < w1; c1 += 32 * TU) {
      unsigned k4[TU];
      load4(c1, k4);
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        bool eq, gt;
        flags_of(c1 + 32 * u + lane, k4[u], &eq, &gt);
        w_eq += __popc(__ballot_sync(0xffffffffu, eq));
      }
    }
    int tot;
    const int eq_before = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? w_eq : 0, sh.scan, &tot), 0);
    int w_k = 0, w_tok = 0;
    long long e2 = eq_before;
    for (long long c1 = w0; c1 < w1; c1 += 32 * TU) {
      unsigned k4[TU];
      load4(c1, k4);
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const long long c0 = c1 + 32 * u;
        bool eq, gt;
        flags_of(c0 + lane, k4[u], &eq, &gt);
        const unsigned eqm = __ballot_sync(0xffffffffu, eq);
        const bool keep = gt || (eq && e2 + __popc(eqm & lt) < need_eq);
        e2 += __popc(eqm);
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        w_k += __popc(km);
        int sz = keep ? csize(c0 + lane) : 0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sz += __shfl_xor_sync(0xffffffffu, sz, o);
        w_tok += sz;
      }
    }
    const int k_before = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? w_k : 0, sh.scan, &tot), 0);
    int tok_total = 0;
    const int tok_before = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? w_tok : 0, sh.scan, &tok_total), 0);
    int kk = k_before, o = tok_before;
    long long e3 = eq_before;
    for (long long c1 = w0; c1 < w1; c1 += 32 * TU) {
      unsigned k4[TU];
      load4(c1, k4);
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const long long c = c1 + 32 * u + lane;
        const unsigned key = k4[u];
        bool eq, gt;
        flags_of(c, key, &eq, &gt);
        const unsigned eqm = __ballot_sync(0xffffffffu, eq);
        const bool keep = gt || (eq && e3 + __popc(eqm & lt) < need_eq);
        e3 += __popc(eqm);
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (V == kCand) {
          if (keep)
            a.cand[(long long)b * K_sel + kk + __popc(km & lt)] =
                ((unsigned long long)key << 32) | (unsigned long long)(~(unsigned)(c + c_base));
          kk += __popc(km);
          continue;
        }
        const int sz = keep ? csize(c) : 0;
        int incl = sz;                                          // inclusive prefix of the kept sizes
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += y;
        }
        if (keep) {
          const int t0 = (int)(c * chunk), oo = o + incl - sz;
          for (int j = 0; j < sz; ++j) {
            ids[oo + j] = t0 + j;
            pos[oo + j] = t0 + j + a.pos0;
            if (out) out[oo + j] = tokens[t0 + j];
          }
        }
        o += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (V != kCand && tid == 0) a.n_kept[b] = tok_total;
    SEL_STAMP(5);
    return;
  }
  for (long long base = 0; base < n_c; base += NT) {
    const long long c = base + tid;
    const unsigned key = c < n_c ? __float_as_uint(cs[c]) : 0u;
    const bool in = c < n_c && (V != kMerge || key != kInvalid);
    const int eq = (in && (key & pmask) == T) ? 1 : 0;
    const int gt = (in && (key & pmask) > T) ? 1 : 0;
    int tot;
    const int eq_rank = block_excl_scan<NT>(eq, sh.scan, &tot) + carry_eq;
    carry_eq += tot;
    const int keep = gt | (eq & (eq_rank < need_eq ? 1 : 0));
    const int slot = block_excl_scan<NT>(keep, sh.scan, &tot);          // index among kept chunks of this tile
    const int nk = tot;
    if (V == kCand) {
      if (keep)
        a.cand[(long long)b * K_sel + carry_k + slot] =
            ((unsigned long long)key << 32) | (unsigned long long)(~(unsigned)(c + c_base));
      carry_k += nk;
      continue;
    }
    int sz = 0;
    if (keep) sz = (int)(((c + 1) * chunk < N ? (c + 1) * chunk : N) - c * chunk);
    int tot2;
    const int off = block_excl_scan<NT>(sz, sh.scan, &tot2) + carry_tok;
    if (keep) {
      sh.kept_c[slot] = (int)c;
      sh.kept_off[slot] = off;
    }
    __syncthreads();
    // one warp per kept chunk: coalesced ids / pos (/ gathered tokens)
    for (int k = warp; k < nk; k += NT / 32) {
      const long long cc = sh.kept_c[k];
      const int t0 = (int)(cc * chunk);
      const int csz = (int)(((cc + 1) * chunk < N ? (cc + 1) * chunk : N) - cc * chunk);
      const int o = sh.kept_off[k];
      for (int j = lane; j < csz; j += 32) {
        ids[o + j] = t0 + j;
        pos[o + j] = t0 + j + a.pos0;
        if (out) out[o + j] = tokens[t0 + j];
      }
    }
    carry_tok += tot2;
    __syncthreads();
  }
  if (V != kCand && tid == 0) a.n_kept[b] = carry_tok;
  SEL_STAMP(5);
}

}  // namespace sel
}  // namespace sp
